#!/usr/bin/env python
"""A small run of every device code path, for compute-sanitizer (one tool per run:
memcheck, racecheck, initcheck, synccheck, profiles/r02_sanitizer_*.txt).

Covers: graph validation and table builders (every table layout, weighted /
unweighted, directed / undirected), the table walker in every mode (default
first-order / node2vec, SUSS-approximated, outlier-folded, partitioned tables),
the counting build, the v3 fenced-search walker, the CDF sampler, the SkipGram pair
kernel and the streamed walks -> SkipGram path, and the host-buffer path.  Every
result is checked against the oracle, so a run that exits 0 also computed the
right walks.  Exit code 0 = all checks passed (the sanitizer adds its own verdict).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2110_06196_b200 as grape  # noqa: E402
from graphgen import tiny_graph, config_graph  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

LAYOUTS = {"auto": None,
           "slim": ({"guide_bytes": 8, "guide_factor": 2}, {"record_bytes": 16}),
           "compact": ({"record_bytes": 16, "guide_bytes": 8, "guide_factor": 1, "hash_h": 6},
                       {"record_bytes": 8, "hash_h": 6})}


def check(name, got, exp):
    got = got.cpu().numpy().view(np.uint32) if torch.is_tensor(got) else got
    if not np.array_equal(got, exp):
        raise SystemExit(f"sanitize_run: {name} differs from the oracle")


def main():
    torch.cuda.set_device(0)
    cases = [tiny_graph(3, 60, 0.08, weighted=True), tiny_graph(4, 50, 0.1, directed=True, weighted=True,
                                                                self_loops=True),
             tiny_graph(5, 70, 0.06, weighted=False), config_graph(2, scale_down=10)]
    for g in cases:
        o = Oracle(*g.numpy())
        starts = np.concatenate([np.arange(g.n), [g.n + 1]]).astype(np.uint32)
        st = torch.as_tensor(starts.view(np.int32)).cuda()
        L = 19
        for lname, lay in LAYOUTS.items():
            layout = None if lay is None else lay[0 if g.w is not None else 1]
            dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, layout=layout)
            for p, q in ((0.5, 2.0), (1.0, 0.25), (1.0, 1.0)):
                e, _ = o.walks(starts, L, mode="node2vec", p=p, q=q, seed=5, base=7)
                check(f"{g.name} {lname} node2vec", grape.walks_node2vec(dg, st, L, p, q, seed=5, walk_id_base=7), e)
            e, _ = o.walks(starts, L, mode="first_order", seed=5)
            check(f"{g.name} {lname} first", grape.walks_first_order(dg, st, L, seed=5), e)
            out, _ = grape.walks_stats(dg, st, L, node2vec=True, p=0.5, q=2.0, seed=5)
            e, _ = o.walks(starts, L, mode="node2vec", p=0.5, q=2.0, seed=5)
            check(f"{g.name} {lname} stats", out, e)
            e, _ = o.walks_approx(starts, L, 3, mode="node2vec", p=0.5, q=2.0, seed=5)
            check(f"{g.name} {lname} approx", grape.walks_approx(dg, st, L, 3, node2vec=True, p=0.5, q=2.0, seed=5), e)
            if not (lname == "compact" and g.w is not None and not g.symmetric):
                e, _ = o.walks_folded(starts, L, p=0.25, q=4.0, seed=5)
                check(f"{g.name} {lname} folded", grape.walks_node2vec_folded(dg, st, L, 0.25, 4.0, seed=5), e)
            e, _ = o.walks_cdf(starts, L, p=0.5, q=2.0, seed=5)
            check(f"{g.name} {lname} cdf", grape.walks_node2vec_cdf(dg, st, L, 0.5, 2.0, seed=5), e)
            w = grape.walks_node2vec(dg, st, L, 0.5, 2.0, seed=5)
            ew, _ = o.walks(starts, L, mode="node2vec", p=0.5, q=2.0, seed=5)
            c, x, ng = grape.skipgram_pairs(dg, w, 2, 3, seed=1)
            ec, ex, en = o.skipgram(ew, 2, 3, seed=1)
            check(f"{g.name} {lname} skipgram", ng, en)
            c2, x2, n2 = grape.walks_skipgram(dg, st, L, 2, 3, node2vec=True, p=0.5, q=2.0, seed=5, pair_seed=1,
                                              chunk_walks=7)
            check(f"{g.name} {lname} streamed", n2, en)
            check(f"{g.name} {lname} streamed centers", c2, ec)
            h = grape.walks_node2vec(dg, torch.as_tensor(starts.view(np.int32)), L, 0.5, 2.0, seed=5)
            check(f"{g.name} {lname} host path", h, ew)
            dg.free()
        # partitioned tables (chunks over 3 owners on this GPU) and the v3 walker
        dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
        dg.partition([0, 0, 0])
        e, _ = o.walks(starts, L, mode="node2vec", p=2.0, q=0.5, seed=6)
        check(f"{g.name} parts", grape.walks_node2vec(dg, st, L, 2.0, 0.5, seed=6), e)
        dg.free()
        dv = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, tables=False)
        check(f"{g.name} v3", grape.walks_node2vec(dv, st, L, 2.0, 0.5, seed=6), e)
        dv.free()
    torch.cuda.synchronize()
    print("sanitize_run: all checks passed")


if __name__ == "__main__":
    main()

"""Tables past 2^32 arcs ("wide": 34-bit arc offsets; DESIGN.md §6 index ranges).

A graph of 4.3e9+ arcs does not fit a test, so the test hook GRAPE_TEST_ARC_BIAS offsets
every row start the walker sees — in the node records and in the records' copy of the
head's row start — by 3·2^32 and moves the walker's table bases back by as much: the
wide walker then runs its 34-bit offset arithmetic (bits 32-33 carried in bits 26-27 of
a record's degree word, u64 row starts in registers, 64-bit floor(start / H) for the
edge hash) on small graphs, and every walk must still equal the oracle's."""
import numpy as np
import pytest
import torch

from graphgen import config_graph, starts_per_node, tiny_graph
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
BIAS = 3 * 2 ** 32   # a multiple of 12: divisible by both edge-hash bucket widths H = 4, 6

LAYOUTS = {"auto": (None, None),
           "slim": ({"guide_bytes": 8, "guide_factor": 2}, {"record_bytes": 16}),
           "compact": ({"record_bytes": 16, "guide_bytes": 8, "guide_factor": 1, "hash_h": 6},
                       {"record_bytes": 8, "hash_h": 6}),
           "fat4": ({"record_bytes": 32, "guide_bytes": 32, "guide_factor": 4, "hash_h": 6}, {"record_bytes": 16,
                                                                                               "hash_h": 6})}


@pytest.fixture()
def grape(monkeypatch):
    monkeypatch.setenv("GRAPE_TEST_ARC_BIAS", str(BIAS))
    import paper_2110_06196_b200 as grape
    return grape


@pytest.mark.parametrize("layout", sorted(LAYOUTS))
@pytest.mark.parametrize("seed,n,dens,directed,weighted", [(1, 60, 0.1, False, True), (2, 80, 0.06, True, True),
                                                          (3, 70, 0.08, False, False), (4, 50, 0.1, True, False)])
def test_wide_offsets_walks_equal_the_oracle(grape, layout, seed, n, dens, directed, weighted):
    g = tiny_graph(2000 + seed, n, dens, directed=directed, weighted=weighted, self_loops=directed)
    lay = LAYOUTS[layout][0 if weighted else 1]
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=not directed, layout=lay)
    assert dg.info["tables"] == 1 and dg.info["wide"] == 1
    o = Oracle(*g.numpy())
    starts = np.concatenate([np.arange(g.n), [g.n + 2]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    for mode, p, q in (("node2vec", 0.5, 2.0), ("node2vec", 2.0, 0.5), ("node2vec", 0.25, 4.0), ("first_order", 1, 1)):
        steps = torch.zeros(1, dtype=torch.int64, device="cuda")
        if mode == "node2vec":
            out = grape.walks_node2vec(dg, st, 33, p, q, seed=9, walk_id_base=7, steps=steps)
        else:
            out = grape.walks_first_order(dg, st, 33, seed=9, walk_id_base=7, steps=steps)
        torch.cuda.synchronize()
        exp, esteps = o.walks(starts, 33, mode=mode, p=p, q=q, seed=9, base=7)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), exp), (mode, p, q)
        assert int(steps.item()) == esteps
    # counting build, SkipGram (reads off[], not the biased starts) on the same graph
    out, stats = grape.walks_stats(dg, st, 20, node2vec=True, p=0.5, q=2.0, seed=3)
    exp, esteps = o.walks(starts, 20, mode="node2vec", p=0.5, q=2.0, seed=3)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), exp) and stats["steps"] == esteps
    c, x, ng = grape.skipgram_pairs(dg, out, 2, 3, seed=1)
    ec, ex, en = o.skipgram(exp, 2, 3, seed=1)
    assert np.array_equal(ng.cpu().numpy().view(np.uint32), en)


def test_wide_graph_full_config_sample(grape):
    """configs[1] scaled down by 2^4 (2.5e6 arcs, fat guide) with 3·2^32-offset rows."""
    g = config_graph(2, scale_down=4)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    assert dg.info["wide"] == 1
    starts = starts_per_node(g.n, 2)
    out = grape.walks_node2vec(dg, starts.cuda(), 40, 0.5, 2.0, seed=42)
    torch.cuda.synchronize()
    o = Oracle(*g.numpy())
    st = starts.numpy().view(np.uint32)
    got = out.cpu().numpy().view(np.uint32)
    rng = np.random.default_rng(0)
    for i in np.unique(rng.integers(0, len(st), 2000)):
        exp, _ = o.walks(st[i:i + 1], 40, mode="node2vec", p=0.5, q=2.0, seed=42, base=int(i))
        assert np.array_equal(got[i], exp[0]), int(i)


def test_wide_graph_modes_refused(grape):
    g = tiny_graph(7, 40, 0.1, weighted=True)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    st = torch.arange(g.n, dtype=torch.int32, device="cuda")
    for call in (lambda: grape.walks_approx(dg, st, 10, 2, p=0.5, q=2.0),
                 lambda: grape.walks_node2vec_cdf(dg, st, 10, 0.5, 2.0),
                 lambda: grape.walks_node2vec_folded(dg, st, 10, 0.25, 4.0)):
        with pytest.raises(grape.GrapeError) as ei:
            call()
        assert ei.value.status == grape.GRAPE_EINVAL
    with pytest.raises(grape.GrapeError):   # the test hook's biased tables are not partitioned
        dg.partition([0, 0])

#!/usr/bin/env python
"""Write tests/golden/kat_modes.json: known-answer rows for the counter conventions of
the §8(f) walk modes and the SkipGram consumer (DESIGN.md §7b f1-c, §7d, §7e f3-c).

Every stored value is computed here by oracle/ alone (the C oracle through
oracle.oracle, cross-checked against the independent Python transliteration
oracle.pyoracle before it is written); nothing comes from the CUDA path.  The rows
freeze the conventions bit for bit: SUSS's bucket draws (counter (wid, s, 2^31 +
b/2), half-blocks), the folded rule's fourth word (o3) and rescaled thresholds,
and SkipGram's slot-keyed negative draws (counter (slot, 0xFFFFFFFF, k/2)).

    python tools/make_kat_modes.py          # rewrites the file
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from oracle.oracle import Oracle, build_oracle  # noqa: E402

PAD = 0xFFFFFFFF


def graphs():
    """Two small graphs written out edge by edge (no generator involved)."""
    # weighted wheel: hub 0 joined to 1..11 (weight = leaf id), rim i - i+1 (weight 2), 1 - 11 closes it
    und = {}
    for i in range(1, 12):
        und[(0, i)] = i
        und[(i, i % 11 + 1)] = 2
    arcs = {}
    for (a, b), w in und.items():
        arcs[(a, b)] = w
        arcs[(b, a)] = w
    wheel = _csr(12, arcs)
    # directed, weighted, with a sink (node 5) and a self-loop (node 3)
    d = {(0, 1): 3, (0, 2): 1, (0, 4): 7, (1, 0): 2, (1, 2): 5, (1, 3): 1, (1, 4): 1, (1, 5): 9, (2, 0): 1,
         (2, 3): 4, (3, 3): 2, (3, 4): 6, (3, 1): 1, (4, 0): 8, (4, 1): 1, (4, 2): 2, (4, 3): 3, (4, 5): 1}
    dirg = _csr(6, d)
    return {"wheel": wheel, "directed6": dirg}


def _csr(n, arcs):
    rows = [[] for _ in range(n)]
    for (a, b), w in sorted(arcs.items()):
        rows[a].append((b, w))
    off, col, w = [0], [], []
    for r in rows:
        for b, ww in r:
            col.append(b)
            w.append(ww)
        off.append(len(col))
    return {"n": n, "off": off, "col": col, "w": w}


def main():
    build_oracle()
    gs = graphs()
    kat = {"source": "tools/make_kat_modes.py: oracle/ only (C oracle, cross-checked with oracle/pyoracle.py). "
                     "Not paper values: they fix the f1 / f2-folded / f3 counter conventions bit for bit "
                     "(DESIGN.md §7b f1-c, §7d, §7e f3-c).",
           "graphs": gs, "approx": [], "folded": [], "skipgram": []}
    for name, g in gs.items():
        o = Oracle(g["n"], np.array(g["off"], dtype=np.uint64), np.array(g["col"], dtype=np.uint32),
                   np.array(g["w"], dtype=np.uint32))
        pg = pyoracle.PyGraph(g["n"], g["off"], g["col"], g["w"])
        starts = list(range(g["n"])) + [g["n"] + 1]
        # SUSS approximated walks, d_T = 3 (the wheel's hub has degree 11, its rim nodes 3)
        for mode, p, q, k, base in (("node2vec", 0.5, 2.0, 3, 0), ("node2vec", 0.25, 4.0, 2, 2 ** 32 - 3),
                                    ("first_order", 1.0, 1.0, 3, 7)):
            out, steps = o.walks_approx(np.array(starts, dtype=np.uint32), 12, k, mode=mode, p=p, q=q, seed=42,
                                        base=base)
            for i, s0 in enumerate(starts):
                row, _ = pg.walk_approx(s0, base + i, 12, k, mode=mode, p=p, q=q, seed=42)
                assert row == out[i].tolist(), (name, mode, i)
            kat["approx"].append({"graph": name, "mode": mode, "p": p, "q": q, "dT": k, "L": 12, "seed": 42,
                                  "base": base, "starts": starts, "rows": out.tolist(), "steps": steps})
        # outlier-folded node2vec (p < min(1, q): the fold applies)
        for p, q, base in ((0.25, 4.0, 0), (0.5, 2.0, 2 ** 40 + 1)):
            out, steps = o.walks_folded(np.array(starts, dtype=np.uint32), 12, p=p, q=q, seed=42, base=base)
            for i, s0 in enumerate(starts):
                row, _ = pg.walk_folded(s0, base + i, 12, p=p, q=q, seed=42)
                assert row == out[i].tolist(), (name, p, q, i)
            kat["folded"].append({"graph": name, "p": p, "q": q, "L": 12, "seed": 42, "base": base,
                                  "starts": starts, "rows": out.tolist(), "steps": steps})
        # SkipGram pairs + negatives of the exact node2vec walks (window 2, K = 3)
        walks, _ = o.walks(np.array(starts[:5], dtype=np.uint32), 6, mode="node2vec", p=0.5, q=2.0, seed=42)
        for win, K, base in ((2, 3, 0), (1, 2, 2 ** 33 + 5)):
            c, x, ng = o.skipgram(walks, win, K, seed=7, base=base)
            pc, px, png = pyoracle.skipgram(pg, walks.tolist(), win, K, seed=7, base=base)
            assert c.tolist() == pc and x.tolist() == px and ng.tolist() == png, (name, win, K)
            kat["skipgram"].append({"graph": name, "walks": walks.tolist(), "window": win, "K": K, "seed": 7,
                                    "base": base, "centers": c.tolist(), "contexts": x.tolist(),
                                    "negatives": ng.tolist()})
    path = os.path.join(ROOT, "tests", "golden", "kat_modes.json")
    with open(path, "w") as f:
        json.dump(kat, f, separators=(",", ":"))
        f.write("\n")
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

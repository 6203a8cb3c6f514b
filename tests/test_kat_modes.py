"""Known-answer rows for the §8(f) mode conventions (tests/golden/kat_modes.json,
written by tools/make_kat_modes.py from oracle/ alone): SUSS approximated walks
(reading f1-c), the outlier-folded rule (§7d) and the SkipGram
consumer's negatives (§7e, reading f3-c).  The CPU tests hold the C oracle and the
Python transliteration to the stored rows (a change to either side's counter
convention fails here, not only their mutual agreement); the GPU tests hold the
CUDA path to the same rows through the C-ABI."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import pyoracle
from oracle.oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KAT = json.load(open(os.path.join(ROOT, "tests", "golden", "kat_modes.json")))


def _graph(name):
    g = KAT["graphs"][name]
    return g, Oracle(g["n"], np.array(g["off"], dtype=np.uint64), np.array(g["col"], dtype=np.uint32),
                     np.array(g["w"], dtype=np.uint32)), pyoracle.PyGraph(g["n"], g["off"], g["col"], g["w"])


def test_kat_modes_cover_the_conventions():
    assert len(KAT["approx"]) == 6 and len(KAT["folded"]) == 4 and len(KAT["skipgram"]) == 4
    # the SUSS cases really sub-sample (some row has degree > d_T) and wide walk ids appear
    for case in KAT["approx"]:
        g = KAT["graphs"][case["graph"]]
        assert max(np.diff(g["off"])) > case["dT"]
    assert any(c["base"] >= 2 ** 32 for c in KAT["folded"])
    assert any(c["base"] >= 2 ** 32 for c in KAT["skipgram"])


@pytest.mark.parametrize("i", range(6))
def test_kat_approx_oracle(i):
    c = KAT["approx"][i]
    g, o, pg = _graph(c["graph"])
    out, steps = o.walks_approx(np.array(c["starts"], dtype=np.uint32), c["L"], c["dT"], mode=c["mode"],
                                p=c["p"], q=c["q"], seed=c["seed"], base=c["base"])
    assert out.tolist() == c["rows"] and steps == c["steps"]
    for j, s0 in enumerate(c["starts"]):
        row, _ = pg.walk_approx(s0, c["base"] + j, c["L"], c["dT"], mode=c["mode"], p=c["p"], q=c["q"],
                                seed=c["seed"])
        assert row == c["rows"][j]


@pytest.mark.parametrize("i", range(4))
def test_kat_folded_oracle(i):
    c = KAT["folded"][i]
    g, o, pg = _graph(c["graph"])
    out, steps = o.walks_folded(np.array(c["starts"], dtype=np.uint32), c["L"], p=c["p"], q=c["q"],
                                seed=c["seed"], base=c["base"])
    assert out.tolist() == c["rows"] and steps == c["steps"]
    for j, s0 in enumerate(c["starts"]):
        row, _ = pg.walk_folded(s0, c["base"] + j, c["L"], p=c["p"], q=c["q"], seed=c["seed"])
        assert row == c["rows"][j]


@pytest.mark.parametrize("i", range(4))
def test_kat_skipgram_oracle(i):
    c = KAT["skipgram"][i]
    g, o, pg = _graph(c["graph"])
    cc, xx, ng = o.skipgram(np.array(c["walks"], dtype=np.uint32), c["window"], c["K"], seed=c["seed"],
                            base=c["base"])
    assert cc.tolist() == c["centers"] and xx.tolist() == c["contexts"] and ng.tolist() == c["negatives"]
    pc, px, png = pyoracle.skipgram(pg, c["walks"], c["window"], c["K"], seed=c["seed"], base=c["base"])
    assert pc == c["centers"] and px == c["contexts"] and png == c["negatives"]


# ---- the CUDA path against the same rows (through the C-ABI)
def _dev(name):
    import paper_2110_06196_b200 as grape
    g = KAT["graphs"][name]
    off = torch.tensor(g["off"], dtype=torch.int64)
    col = torch.tensor(g["col"], dtype=torch.int32)
    w = torch.tensor(g["w"], dtype=torch.int32)
    sym = name == "wheel"
    return grape, grape.graph_from_csr(off, col, w, device=0, symmetric=sym)


@pytest.mark.gpu
def test_kat_modes_gpu():
    for c in KAT["approx"]:
        grape, dg = _dev(c["graph"])
        st = torch.tensor(np.array(c["starts"], dtype=np.uint32).view(np.int32), device="cuda")
        steps = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = grape.walks_approx(dg, st, c["L"], c["dT"], node2vec=c["mode"] == "node2vec", p=c["p"], q=c["q"],
                                 seed=c["seed"], walk_id_base=c["base"], steps=steps)
        torch.cuda.synchronize()
        assert out.cpu().numpy().view(np.uint32).tolist() == c["rows"], c["graph"]
        assert int(steps.item()) == c["steps"]
    for c in KAT["folded"]:
        grape, dg = _dev(c["graph"])
        st = torch.tensor(np.array(c["starts"], dtype=np.uint32).view(np.int32), device="cuda")
        out = grape.walks_node2vec_folded(dg, st, c["L"], c["p"], c["q"], seed=c["seed"], walk_id_base=c["base"])
        torch.cuda.synchronize()
        assert out.cpu().numpy().view(np.uint32).tolist() == c["rows"], c["graph"]
    for c in KAT["skipgram"]:
        grape, dg = _dev(c["graph"])
        walks = torch.tensor(np.array(c["walks"], dtype=np.uint32).view(np.int32), device="cuda")
        cc, xx, ng = grape.skipgram_pairs(dg, walks, c["window"], c["K"], seed=c["seed"], walk_id_base=c["base"])
        torch.cuda.synchronize()
        assert cc.cpu().numpy().view(np.uint32).tolist() == c["centers"]
        assert xx.cpu().numpy().view(np.uint32).tolist() == c["contexts"]
        assert ng.cpu().numpy().view(np.uint32).tolist() == c["negatives"]

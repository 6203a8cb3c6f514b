"""GPU parity of the outlier-folded rejection sampler (
DESIGN.md §7d) through grape_walks_node2vec_folded: every walk bit-identical to
oracle_walks_folded, on every table layout it supports, return-heavy and other
(p, q) settings; its counting build; the identity with the default rule when
p >= min(1, q); configs[1] and configs[4] at full size, sampled."""
import numpy as np
import pytest
import torch

from graphgen import config_graph, config_walks, starts_per_node, tiny_graph
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu

LAYOUTS_W = [None, {"guide_bytes": 8, "guide_factor": 2}, {"record_bytes": 16, "guide_factor": 1, "hash_h": 6}]
LAYOUTS_U = [None, {"record_bytes": 8}]
PQ = [(0.25, 4.0), (0.5, 2.0), (0.3, 1.0), (0.1, 0.5), (2.0, 0.5), (1.0, 1.0)]


@pytest.fixture(scope="module")
def grape():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2110_06196_b200 as grape
    return grape


@pytest.mark.parametrize("seed,n,dens,directed,weighted", [
    (1, 80, 0.06, False, False), (2, 80, 0.06, False, True), (3, 120, 0.05, True, True),
    (4, 60, 0.1, True, False), (5, 200, 0.03, False, True), (6, 30, 0.5, False, True)])
def test_folded_every_walk_bit_exact(grape, seed, n, dens, directed, weighted):
    g = tiny_graph(2000 + seed, n, dens, directed=directed, weighted=weighted, self_loops=directed)
    o = Oracle(*g.numpy())
    starts = np.concatenate([np.arange(g.n), np.arange(g.n)[::-1], [g.n + 1]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    layouts = LAYOUTS_W if weighted else LAYOUTS_U
    for lay in layouts:
        d = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, layout=lay)
        if weighted and directed and lay and lay.get("record_bytes") == 16 and not d.info["weights_symmetric"]:
            with pytest.raises(grape.GrapeError):   # return-arc weights are not kept in 16-B records
                grape.walks_node2vec_folded(d, st, 5, 0.25, 4.0)
            d.free()
            continue
        for p, q in PQ:
            for L in (2, 40):
                exp, esteps = o.walks_folded(starts, L, p=p, q=q, seed=seed, base=7)
                steps = torch.zeros(1, dtype=torch.int64, device="cuda")
                out = grape.walks_node2vec_folded(d, st, L, p, q, seed=seed, walk_id_base=7, steps=steps)
                torch.cuda.synchronize()
                assert np.array_equal(out.cpu().numpy().view(np.uint32), exp), (lay, p, q, L)
                assert int(steps.item()) == esteps
        d.free()


def test_folded_equals_default_when_not_return_heavy_and_stats(grape):
    g = tiny_graph(2100, 150, 0.05, weighted=True)
    d = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    st = torch.arange(g.n, dtype=torch.int32, device="cuda")
    for p, q in [(2.0, 0.5), (1.0, 0.25), (4.0, 1.0)]:
        assert torch.equal(grape.walks_node2vec_folded(d, st, 30, p, q, seed=5),
                           grape.walks_node2vec(d, st, 30, p, q, seed=5))
    plain = grape.walks_node2vec_folded(d, st, 30, 0.25, 4.0, seed=5)
    out, ev = grape.walks_stats(d, st, 30, node2vec=True, p=0.25, q=4.0, seed=5, sampler="folded")
    torch.cuda.synchronize()
    assert torch.equal(out, plain)
    _, esteps, eatt = Oracle(*g.numpy()).walks_folded(st.cpu().numpy().view(np.uint32), 30, p=0.25, q=4.0, seed=5,
                                                      with_attempts=True)
    first = int(np.sum(out.cpu().numpy()[:, 1] != -1))
    assert ev["steps"] == esteps and ev["attempts"] == eatt + first


@pytest.mark.parametrize("k", [2, 5])
def test_full_size_folded_sampled(grape, k):
    wk = config_walks(k)
    g = config_graph(k, device="cuda")
    d = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
    gc = g.to("cpu")
    del g
    torch.cuda.empty_cache()
    W = gc.n * wk["walks_per_node"]
    starts = starts_per_node(gc.n, wk["walks_per_node"], device="cuda")
    out = grape.walks_node2vec_folded(d, starts, wk["L"], wk["p"], wk["q"], seed=wk["seed"])
    torch.cuda.synchronize()
    rng = np.random.default_rng(k + 50)
    sample = np.unique(rng.integers(0, W, 600))
    idx = torch.as_tensor(sample, device="cuda")
    got = out[idx].cpu().numpy().view(np.uint32)
    st_np = starts[idx].cpu().numpy().view(np.uint32)
    del out
    d.free()
    o = Oracle(*gc.numpy())
    for r, i in enumerate(sample):
        exp, _ = o.walks_folded(st_np[r:r + 1], wk["L"], p=wk["p"], q=wk["q"], seed=wk["seed"], base=int(i))
        assert np.array_equal(got[r], exp[0]), int(i)

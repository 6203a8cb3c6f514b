"""The §8(f) f4 table layout (grape_graph_partition): sampling
tables split into power-of-two parts (here all on this one GPU), read by the walker
through its partition map.  Every walk bit-identical to the unpartitioned graph and
to the oracle, on every table layout; the default-rule entry points keep working
(host buffers, counting build, SkipGram); the other modes refuse; configs[1] at full
size in 8 parts."""
import numpy as np
import pytest
import torch

from graphgen import config_graph, config_walks, starts_per_node, tiny_graph
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu

LAYOUTS_W = [None, {"guide_bytes": 8, "guide_factor": 2}, {"record_bytes": 16, "guide_factor": 1}]
LAYOUTS_U = [None, {"record_bytes": 8}]


@pytest.fixture(scope="module")
def grape():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2110_06196_b200 as grape
    return grape


@pytest.mark.parametrize("parts", [2, 3, 8])
@pytest.mark.parametrize("seed,n,dens,directed,weighted", [
    (1, 3000, 0.004, False, True), (2, 3000, 0.004, False, False), (3, 2500, 0.005, True, True)])
def test_partitioned_walks_bit_exact(grape, parts, seed, n, dens, directed, weighted):
    g = tiny_graph(3100 + seed, n, dens, directed=directed, weighted=weighted, self_loops=directed)
    o = Oracle(*g.numpy())
    starts = np.concatenate([np.arange(g.n), [g.n + 1]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    for lay in (LAYOUTS_W if weighted else LAYOUTS_U):
        dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, layout=lay)
        ref = grape.walks_node2vec(dg, st, 25, 0.5, 2.0, seed=seed, walk_id_base=9)
        dg.partition([0] * parts)
        assert dg.info["parts"] == parts and dg.info["tables"] == 1
        for mode, p, q in (("node2vec", 0.5, 2.0), ("node2vec", 2.0, 0.25), ("first_order", 1, 1)):
            steps = torch.zeros(1, dtype=torch.int64, device="cuda")
            if mode == "node2vec":
                out = grape.walks_node2vec(dg, st, 25, p, q, seed=seed, walk_id_base=9, steps=steps)
            else:
                out = grape.walks_first_order(dg, st, 25, seed=seed, walk_id_base=9, steps=steps)
            torch.cuda.synchronize()
            exp, esteps = o.walks(starts, 25, mode=mode, p=p, q=q, seed=seed, base=9)
            assert np.array_equal(out.cpu().numpy().view(np.uint32), exp), (lay, mode, parts)
            assert int(steps.item()) == esteps
        assert torch.equal(grape.walks_node2vec(dg, st, 25, 0.5, 2.0, seed=seed, walk_id_base=9), ref)
        dg.free()


def test_partitioned_entry_points_and_refusals(grape):
    g = tiny_graph(3200, 800, 0.01, weighted=True)
    st = torch.arange(g.n, dtype=torch.int32)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    dev_ref = grape.walks_node2vec(dg, st.cuda(), 30, 0.25, 4.0, seed=3)
    out_ref, ev_ref = grape.walks_stats(dg, st.cuda(), 30, node2vec=True, p=0.25, q=4.0, seed=3)
    c_ref = grape.skipgram_pairs(dg, dev_ref, 3, 2, seed=5)
    dg.partition([0, 0, 0, 0])
    assert torch.equal(grape.walks_node2vec(dg, st, 30, 0.25, 4.0, seed=3), dev_ref.cpu())   # host buffers
    out, ev = grape.walks_stats(dg, st.cuda(), 30, node2vec=True, p=0.25, q=4.0, seed=3)
    assert torch.equal(out, out_ref) and ev == ev_ref
    c = grape.skipgram_pairs(dg, dev_ref, 3, 2, seed=5)
    assert all(torch.equal(a, b) for a, b in zip(c, c_ref))
    for call in (lambda: grape.walks_approx(dg, st.cuda(), 30, 3, p=0.5, q=2.0),
                 lambda: grape.walks_node2vec_cdf(dg, st.cuda(), 30, 0.5, 2.0),
                 lambda: grape.walks_node2vec_folded(dg, st.cuda(), 30, 0.25, 4.0),
                 lambda: dg.partition([0, 0])):
        with pytest.raises(grape.GrapeError) as ei:
            call()
        assert ei.value.status == grape.GRAPE_EINVAL
    with pytest.raises(grape.GrapeError):
        grape.graph_from_csr(g.off, g.col, g.w, device=0, tables=False).partition([0, 0])
    with pytest.raises(grape.GrapeError):
        grape.graph_from_csr(g.off, g.col, g.w, device=0).partition([0, 99])
    dg.free()


def test_cfg2_in_eight_parts(grape):
    """configs[1] at full size, tables in 8 parts: a seeded sample of walks equals the
    unpartitioned graph's (and the oracle's, for a few)."""
    wk = config_walks(2)
    g = config_graph(2, device="cuda")
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    gc = g.to("cpu")
    del g
    torch.cuda.empty_cache()
    rng = np.random.default_rng(8)
    starts = rng.integers(0, gc.n, 200_000).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    ref = grape.walks_node2vec(dg, st, wk["L"], wk["p"], wk["q"], seed=42, walk_id_base=77)
    dg.partition([0] * 8)
    out = grape.walks_node2vec(dg, st, wk["L"], wk["p"], wk["q"], seed=42, walk_id_base=77)
    assert torch.equal(out, ref)
    exp, _ = Oracle(*gc.numpy()).walks(starts[:300], wk["L"], mode="node2vec", p=wk["p"], q=wk["q"],
                                       seed=42, base=77)
    assert np.array_equal(out[:300].cpu().numpy().view(np.uint32), exp)
    dg.free()

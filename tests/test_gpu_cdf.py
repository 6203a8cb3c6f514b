"""GPU parity of the paper's CDF node2vec sampler
through grape_walks_node2vec_cdf: every walk bit-identical to oracle_walks_cdf,
on every table layout, weighted / unweighted / directed graphs (with hubs so
rows span several 32-arc chunks and the no-common-neighbour flags vary)."""
import numpy as np
import pytest
import torch

from graphgen import config_graph, config_walks, starts_per_node, tiny_graph
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu

LAYOUTS_W = [None, {"record_bytes": 16, "guide_factor": 1}, {"record_bytes": 16, "guide_factor": 1, "hash_h": 6}]
LAYOUTS_U = [None, {"record_bytes": 8}]
PQ = [(0.5, 2.0), (0.25, 4.0), (2.0, 0.5), (1.0, 0.25), (4.0, 1.0), (1.0, 1.0)]


@pytest.fixture(scope="module")
def grape():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2110_06196_b200 as grape
    return grape


def _with_hubs(seed, n, dens, directed, weighted):
    g = tiny_graph(seed, n, dens, directed=directed, weighted=weighted, self_loops=directed)
    off, col = g.off.numpy(), g.col.numpy()
    w = None if g.w is None else g.w.numpy()
    src = np.repeat(np.arange(n), np.diff(off))
    arcs = {(int(a), int(b)): (1 if w is None else int(x)) for a, b, x in
            zip(src, col, w if w is not None else np.ones(len(col)))}
    rng = np.random.default_rng(seed)
    for v in range(1, n):
        if rng.random() < 0.7:
            wt = int(rng.integers(1, 90))
            arcs[(0, v)] = wt
            arcs[(v, 0)] = wt if not directed else int(rng.integers(1, 90))
    keys = sorted(arcs)
    o = np.zeros(n + 1, dtype=np.int64)
    for a, _ in keys:
        o[a + 1] += 1
    o = np.cumsum(o)
    c = np.array([b for _, b in keys], dtype=np.int32)
    ww = torch.from_numpy(np.array([arcs[k] for k in keys], dtype=np.int32)) if weighted else None
    from graphgen import CSR
    return CSR(n, torch.from_numpy(o), torch.from_numpy(c), ww, not directed, f"hubs({seed})")


@pytest.mark.parametrize("seed,n,dens,directed,weighted", [
    (1, 90, 0.05, False, False), (2, 90, 0.05, False, True), (3, 120, 0.05, True, True),
    (4, 70, 0.1, True, False), (5, 40, 0.4, False, True)])
def test_cdf_every_walk_bit_exact(grape, seed, n, dens, directed, weighted):
    g = _with_hubs(seed, n, dens, directed, weighted)
    o = Oracle(*g.numpy())
    starts = np.concatenate([np.arange(g.n), np.arange(g.n)[::-1], [g.n + 3]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    for lay in (LAYOUTS_W if weighted else LAYOUTS_U):
        dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, layout=lay)
        for p, q in PQ:
            for L in (1, 2, 33):
                exp, esteps = o.walks_cdf(starts, L, p=p, q=q, seed=seed, base=13)
                steps = torch.zeros(1, dtype=torch.int64, device="cuda")
                out = grape.walks_node2vec_cdf(dg, st, L, p, q, seed=seed, walk_id_base=13, steps=steps)
                torch.cuda.synchronize()
                got = out.cpu().numpy().view(np.uint32)
                assert np.array_equal(got, exp), (lay, p, q, L)
                assert int(steps.item()) == esteps
        dg.free()


def test_cdf_p_q_one_is_first_order_and_host_path(grape):
    g = _with_hubs(7, 150, 0.04, False, True)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    st = torch.arange(g.n, dtype=torch.int32).repeat(2)
    a = grape.walks_node2vec_cdf(dg, st.cuda(), 40, 1.0, 1.0, seed=3)
    b = grape.walks_first_order(dg, st.cuda(), 40, seed=3)
    assert torch.equal(a, b)
    dev = grape.walks_node2vec_cdf(dg, st.cuda(), 40, 0.5, 2.0, seed=3, walk_id_base=5)
    host = grape.walks_node2vec_cdf(dg, st, 40, 0.5, 2.0, seed=3, walk_id_base=5)
    assert torch.equal(dev.cpu(), host)


def test_cdf_needs_tables(grape):
    g = _with_hubs(8, 30, 0.1, False, False)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, tables=False)
    with pytest.raises(grape.GrapeError) as ei:
        grape.walks_node2vec_cdf(dg, torch.arange(g.n, dtype=torch.int32, device="cuda"), 5, 0.5, 2.0)
    assert ei.value.status == grape.GRAPE_EINVAL


def test_cfg1_cdf_every_walk(grape):
    g = config_graph(1)
    starts = starts_per_node(g.n, 1).numpy().view(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
    o = Oracle(*g.numpy())
    exp, esteps = o.walks_cdf(starts, 32, p=0.5, q=2.0, seed=42)
    out = grape.walks_node2vec_cdf(dg, st, 32, 0.5, 2.0, seed=42)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), exp)


def test_cfg2_cdf_sampled(grape):
    """configs[1] graph at full size, a seeded sample of walks (shortened to L = 20:
    the oracle's CDF step costs O(deg v * log deg t))."""
    g = config_graph(2, device="cuda")
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    gc = g.to("cpu")
    del g
    rng = np.random.default_rng(2)
    starts = rng.integers(0, gc.n, 300).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    out = grape.walks_node2vec_cdf(dg, st, 20, 0.5, 2.0, seed=42, walk_id_base=1000)
    torch.cuda.synchronize()
    exp, _ = Oracle(*gc.numpy()).walks_cdf(starts, 20, p=0.5, q=2.0, seed=42, base=1000)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), exp)

"""GPU parity of the approximated walks (SUSS sub-sampling, SURVEY §8(f) row f1;
P:513-520, Fig. 3) through grape_walks_approx: every walk bit-identical to the
oracle's oracle_walks_approx, on every table layout, weighted / unweighted /
directed graphs with hubs, thresholds from 1 to above the maximum degree."""
import numpy as np
import pytest
import torch

from graphgen import config_graph, config_walks, starts_per_node, tiny_graph
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu

LAYOUTS_W = [None, {"record_bytes": 32, "guide_bytes": 8, "guide_factor": 1},
             {"record_bytes": 16, "guide_factor": 2}, {"record_bytes": 16, "guide_factor": 1, "hash_h": 6}]
LAYOUTS_U = [None, {"record_bytes": 8}]
SETTINGS = [("first_order", 1.0, 1.0), ("node2vec", 0.5, 2.0), ("node2vec", 0.25, 4.0), ("node2vec", 2.0, 0.5),
            ("node2vec", 1.0, 0.25)]


@pytest.fixture(scope="module")
def grape():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2110_06196_b200 as grape
    return grape


def _hub_graph(seed, n, dens, directed, weighted):
    """tiny_graph plus two hubs adjacent to most nodes (degrees >> the thresholds)."""
    g = tiny_graph(seed, n, dens, directed=directed, weighted=weighted, self_loops=directed)
    off, col = g.off.numpy(), g.col.numpy()
    w = None if g.w is None else g.w.numpy()
    src = np.repeat(np.arange(n), np.diff(off))
    arcs = {(int(a), int(b)): (1 if w is None else int(x)) for a, b, x in
            zip(src, col, w if w is not None else np.ones(len(col)))}
    rng = np.random.default_rng(seed)
    for h in (0, 1):
        for v in range(2, n):
            if rng.random() < 0.8:
                wt = int(rng.integers(1, 50))
                arcs[(h, v)] = wt
                arcs[(v, h)] = wt if not directed else int(rng.integers(1, 50))
    keys = sorted(arcs)
    o = np.zeros(n + 1, dtype=np.int64)
    for a, _ in keys:
        o[a + 1] += 1
    o = np.cumsum(o)
    c = np.array([b for _, b in keys], dtype=np.int32)
    ww = np.array([arcs[k] for k in keys], dtype=np.int32) if weighted else None
    from graphgen import CSR
    return CSR(n, torch.from_numpy(o), torch.from_numpy(c), None if ww is None else torch.from_numpy(ww),
               not directed, f"hub({seed})")


def _run(grape, dg, st, L, k, mode, p, q, seed, base):
    steps = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = grape.walks_approx(dg, st, L, k, node2vec=mode == "node2vec", p=p, q=q, seed=seed,
                             walk_id_base=base, steps=steps)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32), int(steps.item())


@pytest.mark.parametrize("seed,n,dens,directed,weighted", [
    (1, 80, 0.05, False, False), (2, 80, 0.05, False, True), (3, 120, 0.04, True, True),
    (4, 60, 0.1, True, False), (5, 200, 0.02, False, True)])
def test_approx_every_walk_bit_exact(grape, seed, n, dens, directed, weighted):
    g = _hub_graph(seed, n, dens, directed, weighted)
    o = Oracle(*g.numpy())
    maxdeg = int(np.max(np.diff(g.off.numpy())))
    assert maxdeg > 40
    starts = np.concatenate([np.arange(g.n), np.arange(g.n)[::-1], [g.n + 5]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    for lay in (LAYOUTS_W if weighted else LAYOUTS_U):
        dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, layout=lay)
        for k in (1, 2, 5, 17, maxdeg - 1, maxdeg):
            for mode, p, q in SETTINGS:
                exp, esteps = o.walks_approx(starts, 24, k, mode=mode, p=p, q=q, seed=seed, base=5)
                got, steps = _run(grape, dg, st, 24, k, mode, p, q, seed, 5)
                assert np.array_equal(got, exp), (lay, k, mode, p, q)
                assert steps == esteps
        dg.free()


def test_threshold_at_or_above_max_degree_is_exact(grape):
    g = _hub_graph(9, 100, 0.05, False, True)
    maxdeg = int(np.max(np.diff(g.off.numpy())))
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    st = torch.arange(g.n, dtype=torch.int32, device="cuda")
    exact = grape.walks_node2vec(dg, st, 30, 0.5, 2.0, seed=4)
    for k in (0, maxdeg, maxdeg + 10):
        ap = grape.walks_approx(dg, st, 30, k, node2vec=True, p=0.5, q=2.0, seed=4)
        assert torch.equal(exact, ap)
    assert not torch.equal(exact, grape.walks_approx(dg, st, 30, 3, node2vec=True, p=0.5, q=2.0, seed=4))


def test_approx_host_buffers_and_sharding(grape):
    g = _hub_graph(11, 150, 0.03, False, True)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    st = torch.arange(g.n, dtype=torch.int32).repeat(3)
    dev = grape.walks_approx(dg, st.cuda(), 20, 4, p=0.5, q=2.0, seed=2, walk_id_base=9)
    host = grape.walks_approx(dg, st, 20, 4, p=0.5, q=2.0, seed=2, walk_id_base=9)
    assert torch.equal(dev.cpu(), host)
    W = st.numel()
    parts = [grape.walks_approx(dg, st[lo:lo + 100].cuda(), 20, 4, p=0.5, q=2.0, seed=2, walk_id_base=9 + lo)
             for lo in range(0, W, 100)]
    assert torch.equal(torch.cat(parts).cpu(), host)


def test_approx_needs_tables(grape):
    g = _hub_graph(12, 60, 0.05, False, False)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, tables=False)
    st = torch.arange(g.n, dtype=torch.int32, device="cuda")
    with pytest.raises(grape.GrapeError) as ei:
        grape.walks_approx(dg, st, 10, 3, p=0.5, q=2.0)
    assert ei.value.status == grape.GRAPE_EINVAL
    # a threshold no row exceeds needs no tables (exact walks)
    big = grape.walks_approx(dg, st, 10, 10 ** 6, p=0.5, q=2.0)
    assert torch.equal(big, grape.walks_node2vec(dg, st, 10, 0.5, 2.0))


@pytest.mark.parametrize("k", [10, 100])
def test_cfg1_approx_every_walk(grape, k):
    """configs[0] graph (max degree ~1.8k): node2vec and first order, d_T = 10 (the
    paper's STRING PPI setting) and 100, every walk."""
    g = config_graph(1)
    wk = config_walks(1)
    starts = starts_per_node(g.n, 1).numpy().view(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
    o = Oracle(*g.numpy())
    for mode, p, q in [("first_order", 1, 1), ("node2vec", 1.0, 0.25)]:
        exp, esteps = o.walks_approx(starts, wk["L"], k, mode=mode, p=p, q=q, seed=42)
        got, steps = _run(grape, dg, st, wk["L"], k, mode, p, q, 42, 0)
        assert np.array_equal(got, exp) and steps == esteps


@pytest.mark.parametrize("k,dT", [(2, 10), (3, 10)])
def test_full_size_config_approx_sampled(grape, k, dT):
    """configs[1] / configs[2] at full size, approximated with d_T = 10 in bench.py's
    launch configuration (one call over all walks): a seeded sample of walks plus the
    walks from the 20 highest-degree nodes, recomputed by the oracle one by one."""
    wk = config_walks(k)
    g = config_graph(k, device="cuda")
    torch.cuda.empty_cache()
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
    deg = g.off[1:] - g.off[:-1]
    hubs = torch.topk(deg, 20).indices.cpu().numpy()
    gc = g.to("cpu")
    del g, deg
    torch.cuda.empty_cache()
    starts = starts_per_node(gc.n, wk["walks_per_node"], device="cuda")
    steps = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = grape.walks_approx(dg, starts, wk["L"], dT, node2vec=True, p=wk["p"], q=wk["q"], seed=wk["seed"],
                             steps=steps)
    torch.cuda.synchronize()
    W = starts.numel()
    rng = np.random.default_rng(100 + k)
    sample = np.unique(np.concatenate([rng.integers(0, W, 400), hubs]))
    idx = torch.as_tensor(sample, device="cuda")
    got = out[idx].cpu().numpy().view(np.uint32)
    st_np = starts[idx].cpu().numpy().view(np.uint32)
    del out
    dg.free()
    o = Oracle(*gc.numpy())
    for r, i in enumerate(sample):
        exp, _ = o.walks_approx(st_np[r:r + 1], wk["L"], dT, mode="node2vec", p=wk["p"], q=wk["q"],
                                seed=wk["seed"], base=int(i))
        assert np.array_equal(got[r], exp[0]), int(i)

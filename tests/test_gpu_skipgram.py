"""GPU parity of the SkipGram consumer through
grape_skipgram_pairs: centers, contexts and every negative bit-identical to
oracle_skipgram on walk matrices the GPU walker produced (ragged PAD suffixes,
isolated starts, bad starts), several windows / negative counts, shard slices;
configs[1] at full graph size on a batch of walks, sampled slots."""
import numpy as np
import pytest
import torch

from graphgen import CSR, config_graph, config_walks, starts_per_node, tiny_graph
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def grape():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2110_06196_b200 as grape
    return grape


def _with_isolated(seed, n, dens, directed):
    g = tiny_graph(seed, n, dens, directed=directed, weighted=True, self_loops=False)
    n0, off0, col0, w0 = g.numpy()
    rng = np.random.default_rng(seed)
    N = n0 + n0 // 3
    ids = np.sort(rng.choice(N, n0, replace=False))
    deg = np.zeros(N, dtype=np.int64)
    deg[ids] = np.diff(off0.astype(np.int64))
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    col = ids[col0.astype(np.int64)].astype(np.int32)
    return CSR(N, torch.from_numpy(off), torch.from_numpy(col), torch.from_numpy(w0.astype(np.int32)),
               not directed, f"iso({seed})")


@pytest.mark.parametrize("seed,directed", [(1, False), (2, True), (3, False)])
@pytest.mark.parametrize("window,K", [(1, 0), (2, 3), (5, 5), (9, 1)])
def test_skipgram_bit_exact(grape, seed, directed, window, K):
    g = _with_isolated(500 + seed, 120, 0.05, directed)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
    o = Oracle(*g.numpy())
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, g.n + 3, 300).astype(np.uint32)
    L = 13
    walks = grape.walks_node2vec(dg, torch.as_tensor(starts.view(np.int32)).cuda(), L, 0.5, 2.0, seed=seed,
                                 walk_id_base=40)
    c, x, ng = grape.skipgram_pairs(dg, walks, window, K, seed=seed + 9, walk_id_base=40)
    torch.cuda.synchronize()
    wn = walks.cpu().numpy().view(np.uint32)
    ec, ex, eng = o.skipgram(wn, window, K, seed=seed + 9, base=40)
    assert np.array_equal(c.cpu().numpy().view(np.uint32), ec)
    assert np.array_equal(x.cpu().numpy().view(np.uint32), ex)
    assert np.array_equal(ng.cpu().numpy().view(np.uint32), eng)
    dg.free()


def test_skipgram_shards_and_errors(grape):
    g = _with_isolated(77, 90, 0.06, False)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    st = starts_per_node(g.n, 2).cuda()
    walks = grape.walks_first_order(dg, st, 9, seed=4)
    c, x, ng = grape.skipgram_pairs(dg, walks, 3, 4, seed=1)
    per = 9 * 6
    W = walks.shape[0]
    for a, b in ((0, 17), (17, 18), (18, W)):
        cs, xs, ns = grape.skipgram_pairs(dg, walks[a:b], 3, 4, seed=1, walk_id_base=a)
        assert torch.equal(cs, c[a * per:b * per]) and torch.equal(xs, x[a * per:b * per])
        assert torch.equal(ns, ng[a * per:b * per])
    with pytest.raises(grape.GrapeError):
        grape.skipgram_pairs(dg, walks, 0, 1)
    # a graph without arcs: every slot invalid
    e = CSR(4, torch.zeros(5, dtype=torch.int64), torch.zeros(0, dtype=torch.int32), None, True)
    de = grape.graph_from_csr(e.off, e.col, None, device=0, symmetric=True)
    we = grape.walks_first_order(de, torch.arange(4, dtype=torch.int32, device="cuda"), 3)
    c0, x0, n0 = grape.skipgram_pairs(de, we, 2, 2)
    assert bool((c0 == -1).all() and (x0 == -1).all() and (n0 == -1).all())


def test_cfg2_batch_sampled(grape):
    """configs[1]'s graph at full size, a batch of 2e5 of its walks (bench.py --skipgram's
    shape, window 5, 5 negatives); 3000 sampled slots against the oracle."""
    wk = config_walks(2)
    g = config_graph(2, device="cuda")
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    gc = g.to("cpu")
    del g
    B = 200_000
    st = starts_per_node(gc.n, wk["walks_per_node"], device="cuda")[:B]
    walks = grape.walks_node2vec(dg, st, wk["L"], wk["p"], wk["q"], seed=wk["seed"])
    c, x, ng = grape.skipgram_pairs(dg, walks, 5, 5, seed=11)
    torch.cuda.synchronize()
    S = c.numel()
    rng = np.random.default_rng(3)
    slots = np.unique(rng.integers(0, S, 3000))
    per = wk["L"] * 10
    o = Oracle(*gc.numpy())
    wn = walks.cpu().numpy().view(np.uint32)
    cn, xn, nn = (t.cpu().numpy().view(np.uint32) for t in (c, x, ng))
    for p in slots:
        r = int(p) // per
        ec, ex, eng = o.skipgram(wn[r:r + 1], 5, 5, seed=11, base=r)
        q = int(p) - r * per
        assert cn[p] == ec[q] and xn[p] == ex[q] and np.array_equal(nn[p], eng[q]), int(p)
    # the law of the negatives at scale: mean out-degree of negatives = E[deg^2]/E[deg]
    deg = np.diff(gc.off.numpy())
    neg = nn[nn != 0xFFFFFFFF][:2_000_000].astype(np.int64)
    want = float((deg.astype(np.float64) ** 2).sum() / deg.sum())
    got = float(deg[neg].mean())
    assert abs(got - want) / want < 0.02


@pytest.mark.parametrize("seed,directed", [(11, False), (12, True)])
@pytest.mark.parametrize("mode,p,q", [("node2vec", 0.5, 2.0), ("first_order", 1.0, 1.0), ("node2vec", 0.25, 4.0)])
@pytest.mark.parametrize("chunk", [1, 7, 100, 0])
def test_walks_skipgram_streamed_equals_two_calls(grape, seed, directed, mode, p, q, chunk):
    """grape_walks_skipgram (walks streamed chunk by chunk into the pair kernel, no walk
    matrix) == grape_walks_* then grape_skipgram_pairs, bit for bit, and == the oracle;
    chunk sizes of 1, 7, 100 rows and the automatic one; the step counter adds up."""
    g = _with_isolated(900 + seed, 150, 0.04, directed)
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=not directed)
    starts = np.concatenate([np.arange(g.n), [g.n + 3], np.arange(g.n)[::-1]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    L, win, K, base = 17, 3, 4, 2 ** 32 - 40
    n2v = mode == "node2vec"
    s1 = torch.zeros(1, dtype=torch.int64, device="cuda")
    s2 = torch.zeros(1, dtype=torch.int64, device="cuda")
    if n2v:
        walks = grape.walks_node2vec(dg, st, L, p, q, seed=42, walk_id_base=base, steps=s1)
    else:
        walks = grape.walks_first_order(dg, st, L, seed=42, walk_id_base=base, steps=s1)
    c1, x1, n1 = grape.skipgram_pairs(dg, walks, win, K, seed=9, walk_id_base=base)
    c2, x2, n2 = grape.walks_skipgram(dg, st, L, win, K, node2vec=n2v, p=p, q=q, seed=42, pair_seed=9,
                                      walk_id_base=base, steps=s2, chunk_walks=chunk)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2) and torch.equal(x1, x2) and torch.equal(n1, n2)
    assert int(s1.item()) == int(s2.item())
    o = Oracle(*g.numpy())
    ew, _ = o.walks(starts, L, mode=mode, p=p, q=q, seed=42, base=base)
    ec, ex, en = o.skipgram(ew, win, K, seed=9, base=base)
    assert np.array_equal(c2.cpu().numpy().view(np.uint32), ec)
    assert np.array_equal(x2.cpu().numpy().view(np.uint32), ex)
    assert np.array_equal(n2.cpu().numpy().view(np.uint32), en)

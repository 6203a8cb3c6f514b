"""GPU parity of the v4 (sampling-table) walker on graphs built to stress its
tables: guide buckets holding many proposal boundaries
(split scans over several record sectors), hub rows whose edge-hash probes
cross sectors and wrap around, complete graphs (every non-return proposal is a
neighbour of t), asymmetric weights (the return interval is unknown after a
return), and directed graphs with reciprocal arcs.  Every walk is compared
with the oracle bit for bit, and with the v3 walker (GRAPE_NO_TABLES)."""
import numpy as np
import pytest
import torch

from graphgen import CSR
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu

PAD = 0xFFFFFFFF
SETTINGS = [("first_order", 1.0, 1.0), ("node2vec", 0.5, 2.0), ("node2vec", 0.25, 4.0),
            ("node2vec", 1.0, 0.25), ("node2vec", 2.0, 0.5), ("node2vec", 4.0, 1.0)]


@pytest.fixture(scope="module")
def grape():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2110_06196_b200 as grape
    return grape


def _csr(n, src, dst, w=None, symmetric=False, name="stress"):
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off)
    wt = None if w is None else torch.from_numpy(np.asarray(w, dtype=np.int64)[order].astype(np.int32))
    return CSR(n, torch.from_numpy(off), torch.from_numpy(dst.astype(np.int32)), wt, symmetric, name)


def _undirected(n, pairs, wfun=None, asym=False, seed=0):
    a = np.array([p[0] for p in pairs], dtype=np.int64)
    b = np.array([p[1] for p in pairs], dtype=np.int64)
    src = np.concatenate([a, b])
    dst = np.concatenate([b, a])
    w = None
    if wfun is not None:
        rng = np.random.default_rng(seed)
        wu = wfun(rng, len(a))
        w = np.concatenate([wu, wfun(rng, len(a)) if asym else wu])
    return _csr(n, src, dst, w, symmetric=True)


def _check_all(grape, g, L=48, seeds=(3,), settings=SETTINGS, expect_wsym=None):
    o = Oracle(*g.numpy())
    starts = np.concatenate([np.arange(g.n), np.arange(g.n)[::-1], [g.n]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    d4 = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
    d3 = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, tables=False)
    assert d4.info["tables"] == 1 and d3.info["tables"] == 0
    assert d4.info["table_bytes"] > 0 and d3.info["table_bytes"] == 0
    if expect_wsym is not None:
        assert d4.info["weights_symmetric"] == int(expect_wsym)
    assert d4.info["guide_factor"] == (4 if g.w is not None else 0)
    for seed in seeds:
        for mode, p, q in settings:
            exp, esteps = o.walks(starts, L, mode=mode, p=p, q=q, seed=seed, base=11)
            for dg in (d4, d3):
                steps = torch.zeros(1, dtype=torch.int64, device="cuda")
                if mode == "first_order":
                    out = grape.walks_first_order(dg, st, L, seed=seed, walk_id_base=11, steps=steps)
                else:
                    out = grape.walks_node2vec(dg, st, L, p, q, seed=seed, walk_id_base=11, steps=steps)
                torch.cuda.synchronize()
                got = out.cpu().numpy().view(np.uint32)
                assert np.array_equal(got, exp), (mode, p, q, seed, dg.info["tables"])
                assert int(steps.item()) == esteps
    d4.free()
    d3.free()


def test_guide_split_buckets_heavy_tailed_weights(grape):
    """Weights 1 or 10^6: the light arcs of a row all fall into one or two guide
    buckets, so a proposal there scans several record sectors."""
    rng = np.random.default_rng(1)
    n = 150
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.4]
    g = _undirected(n, pairs, lambda r, k: np.where(r.random(k) < 0.1, 10 ** 6, 1))
    _check_all(grape, g, seeds=(3, 4), expect_wsym=True)


def test_asymmetric_weights_on_undirected_structure(grape):
    """Each direction of an edge has its own weight: the interval of an arc taken
    forward is not known from its reverse (weights_symmetric = 0)."""
    rng = np.random.default_rng(2)
    n = 120
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.15]
    g = _undirected(n, pairs, lambda r, k: r.integers(1, 1000, k), asym=True)
    _check_all(grape, g, expect_wsym=False)


def test_hub_rows_edge_hash(grape):
    """A hub adjacent to every node plus a sparse random layer: membership tests
    against the hub's 2*deg-slot set and probe runs that cross sectors / wrap."""
    rng = np.random.default_rng(3)
    n = 3000
    pairs = [(0, j) for j in range(1, n)]
    extra = set()
    while len(extra) < 6000:
        a, b = sorted(rng.integers(1, n, 2))
        if a != b:
            extra.add((int(a), int(b)))
    pairs += sorted(extra)
    for weighted in (False, True):
        g = _undirected(n, pairs, (lambda r, k: r.integers(1, 100, k)) if weighted else None)
        _check_all(grape, g, L=40, settings=SETTINGS[1:4])


@pytest.mark.parametrize("k", [2, 9, 33])
def test_complete_graphs(grape, k):
    pairs = [(i, j) for i in range(k) for j in range(i + 1, k)]
    _check_all(grape, _undirected(k, pairs), L=30)
    _check_all(grape, _undirected(k, pairs, lambda r, m: r.integers(1, 7, m)), L=30)


def test_directed_reciprocal_arcs_with_self_loops(grape):
    """Directed graph where about half the arcs have a reverse arc (with a
    different weight) and some nodes have self-loops or no out-arcs."""
    rng = np.random.default_rng(4)
    n = 400
    src, dst = [], []
    for _ in range(3000):
        a, b = rng.integers(0, n, 2)
        src.append(a); dst.append(b)
        if rng.random() < 0.5:
            src.append(b); dst.append(a)
    key = np.unique(np.array(src, dtype=np.int64) * n + np.array(dst, dtype=np.int64))
    s, d = key // n, key % n
    keep = ~np.isin(s, np.arange(0, n, 37))   # some sinks
    s, d = s[keep], d[keep]
    w = rng.integers(1, 50, len(s))
    _check_all(grape, _csr(n, s, d, w), L=40)
    _check_all(grape, _csr(n, s, d), L=40)


def test_single_arc_rows_and_long_walks(grape):
    """Paths and a cycle: deg-1 rows skip the guide; L=300 keeps returns chaining."""
    n = 50
    pairs = [(i, i + 1) for i in range(n - 1)] + [(n - 1, 0)]
    _check_all(grape, _undirected(n, pairs, lambda r, k: r.integers(1, 5, k)), L=300)
    path = [(i, i + 1) for i in range(9)]
    _check_all(grape, _undirected(10, path), L=300)

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

from graphgen import CSR, tiny_graph
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


LAYOUTS_W = [None, {"guide_bytes": 32, "guide_factor": 1}, {"guide_bytes": 8, "guide_factor": 4},
             {"guide_bytes": 32, "guide_factor": 8},
             {"record_bytes": 16, "guide_factor": 2}, {"record_bytes": 16, "guide_factor": 1, "hash_h": 6}]
LAYOUTS_U = [None, {"record_bytes": 8}, {"record_bytes": 16, "hash_h": 6}]


def _check_all(grape, g, L=48, seeds=(3,), settings=SETTINGS, expect_wsym=None):
    """Every walk of every setting on every table layout (and the v3 walker) == oracle."""
    o = Oracle(*g.numpy())
    starts = np.concatenate([np.arange(g.n), np.arange(g.n)[::-1], [g.n]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    graphs = []
    for lay in (LAYOUTS_W if g.w is not None else LAYOUTS_U):
        d = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, layout=lay)
        assert d.info["tables"] == 1 and d.info["table_bytes"] > 0
        for k, v in (lay or {}).items():
            assert d.info[k] == v, (k, d.info)
        if lay is None and g.w is not None:   # small graph: the richest layout
            assert (d.info["record_bytes"], d.info["guide_bytes"], d.info["guide_factor"]) == (32, 32, 16)
        if expect_wsym is not None:
            assert d.info["weights_symmetric"] == int(expect_wsym)
        graphs.append(d)
    d3 = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, tables=False)
    assert d3.info["tables"] == 0 and d3.info["table_bytes"] == 0
    graphs.append(d3)
    for seed in seeds:
        for mode, p, q in settings:
            exp, esteps = o.walks(starts, L, mode=mode, p=p, q=q, seed=seed, base=11)
            for dg in graphs:
                steps = torch.zeros(1, dtype=torch.int64, device="cuda")
                if mode == "first_order":
                    out = grape.walks_first_order(dg, st, L, seed=seed, walk_id_base=11, steps=steps)
                else:
                    out = grape.walks_node2vec(dg, st, L, p, q, seed=seed, walk_id_base=11, steps=steps)
                torch.cuda.synchronize()
                got = out.cpu().numpy().view(np.uint32)
                assert np.array_equal(got, exp), (mode, p, q, seed, dg.info)
                assert int(steps.item()) == esteps
    for d in graphs:
        d.free()


def test_layout_options_rejected_or_enforced(grape):
    g = _undirected(20, [(i, i + 1) for i in range(19)] + [(0, 10), (3, 17)], lambda r, k: r.integers(1, 9, k))
    for bad in ({"record_bytes": 8}, {"guide_bytes": 16}, {"guide_factor": 3}, {"hash_h": 5},
                {"record_bytes": 16, "guide_bytes": 32}):
        with pytest.raises(grape.GrapeError) as ei:
            grape.graph_from_csr(g.off, g.col, g.w, device=0, layout=bad)
        assert ei.value.status == grape.GRAPE_EINVAL
    with pytest.raises(grape.GrapeError) as ei:   # a forced layout that cannot fit the budget
        grape.graph_from_csr(g.off, g.col, g.w, device=0, layout={"record_bytes": 32, "table_budget_bytes": 64})
    assert ei.value.status == grape.GRAPE_ENOMEM
    tiny = grape.graph_from_csr(g.off, g.col, g.w, device=0, layout={"table_budget_bytes": 64})
    assert tiny.info["tables"] == 0   # automatic layout that does not fit: v3 walker
    u = _undirected(20, [(0, 1), (1, 2)])
    with pytest.raises(grape.GrapeError):
        grape.graph_from_csr(u.off, u.col, None, device=0, layout={"guide_factor": 2})


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


def test_random_graphs_random_layouts(grape):
    """60 seeded random cases: graph shape, weights, direction, hub, layout, (p, q),
    walk length, walk-id base and seed all drawn at random; every walk == oracle."""
    rng = np.random.default_rng(2026)
    for case in range(60):
        n = int(rng.integers(2, 160))
        dens = float(rng.uniform(0.0, 0.5))
        directed = bool(rng.integers(0, 2))
        weighted = bool(rng.integers(0, 2))
        g = tiny_graph(5000 + case, n, dens, directed=directed, weighted=weighted, self_loops=directed,
                       max_w=int(rng.choice([3, 100, 60000])))
        lay = (LAYOUTS_W if weighted else LAYOUTS_U)[int(rng.integers(0, len(LAYOUTS_W if weighted else LAYOUTS_U)))]
        p = float(rng.choice([0.25, 0.5, 1.0, 2.0, 4.0, 0.3, 7.0]))
        q = float(rng.choice([0.25, 0.5, 1.0, 2.0, 4.0, 0.3, 7.0]))
        L = int(rng.integers(1, 70))
        seed = int(rng.integers(0, 2 ** 63))
        base = int(rng.integers(0, 2 ** 40))
        starts = rng.integers(0, n + 2, int(rng.integers(1, 3 * n + 2))).astype(np.uint32)
        try:
            d = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric, layout=lay)
        except grape.GrapeError as e:   # a forced layout can be invalid for an edge-less graph
            assert g.m == 0, e
            continue
        exp, esteps = Oracle(*g.numpy()).walks(starts, L, mode="node2vec", p=p, q=q, seed=seed, base=base)
        steps = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = grape.walks_node2vec(d, torch.as_tensor(starts.view(np.int32)).cuda(), L, p, q, seed=seed,
                                   walk_id_base=base, steps=steps)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), exp), (case, n, dens, directed, weighted, lay, p, q)
        assert int(steps.item()) == esteps
        d.free()

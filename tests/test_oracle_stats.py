"""Statistical / closed-form pins of the oracle against what the PAPER fixes.

The paper defines the walks by their law: pi_vx = alpha_pq(t,x) w_vx
(§4.3.1 Eq.1; alpha via x == t and x in N(t)) and the
weighted first-order law w_vx / sum w.  These tests draw many
steps / walks from the oracle and compare them with exact laws computed here
from those formulas (Fractions), or with closed forms derived by hand for
path, star and triangle graphs.  All seeds are fixed, so the tests are
deterministic; thresholds are set so that a correct sampler passes with
overwhelming margin and each mutant below fails.
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

from oracle import pyoracle
from oracle.oracle import Oracle
from graphgen import tiny_graph

HERE = os.path.dirname(os.path.abspath(__file__))
LAWS = json.load(open(os.path.join(HERE, "golden", "paper_laws.json")))
P_MIN = 1e-6   # per-test chi-square p-value floor for a correct sampler (fixed seeds)


def _chi2_p(counts, probs):
    counts = np.asarray(counts, dtype=np.float64)
    exp = np.asarray([float(p) for p in probs]) * counts.sum()
    if len(counts) == 1:
        return 1.0 if counts[0] == exp[0] else 0.0
    return stats.chisquare(counts, exp).pvalue


def _graph_from_edges(n, edges, weights=None):
    arcs = {}
    for a, b in edges:
        wv = 1 if weights is None else weights[f"{min(a, b)}-{max(a, b)}"]
        arcs[(a, b)] = wv
        arcs[(b, a)] = wv
    keys = sorted(arcs)
    off = np.zeros(n + 1, dtype=np.uint64)
    for a, _ in keys:
        off[a + 1] += 1
    off = np.cumsum(off).astype(np.uint64)
    col = np.array([b for _, b in keys], dtype=np.uint32)
    w = None if weights is None else np.array([arcs[k] for k in keys], dtype=np.uint32)
    return n, off, col, w


# --------------------------------------------------------------------------- first order
@pytest.mark.parametrize("case", LAWS["first_order"], ids=lambda c: c["cite"][:6])
def test_first_order_weighted_law(case):
    """Star centre 0 with weights w_i: P(leaf i) = w_i / sum w."""
    k = len(case["weights"])
    off = np.array([0, k] + [k] * k, dtype=np.uint64)
    col = np.arange(1, k + 1, dtype=np.uint32)
    o = Oracle(k + 1, off, col, np.array(case["weights"], dtype=np.uint32))
    N = 1_000_000
    x = o.first_order_steps(0, 1, 0, N)
    counts = np.bincount(x - 1, minlength=k)
    probs = [Fraction(p) for p in case["probs"]]
    assert _chi2_p(counts, probs) > P_MIN
    assert np.max(np.abs(counts / N - np.array([float(p) for p in probs]))) < 0.005   # S:229 tolerance


def test_first_order_unweighted_uniform_star():
    """Unweighted step = uniform over N(v) (S:236 star example)."""
    k = 37
    off = np.array([0, k] + [k] * k, dtype=np.uint64)
    o = Oracle(k + 1, off, np.arange(1, k + 1, dtype=np.uint32), None)
    x = o.first_order_steps(0, 3, 17, 1_000_000)
    counts = np.bincount(x - 1, minlength=k)
    assert _chi2_p(counts, [Fraction(1, k)] * k) > P_MIN


# --------------------------------------------------------------------------- node2vec
@pytest.mark.parametrize("case", LAWS["node2vec"], ids=["S246_unweighted", "S246_weighted"])
def test_node2vec_paper_example(case):
    n, off, col, w = _graph_from_edges(case["n"], case["edges"], case["weights"])
    o = Oracle(n, off, col, w)
    N = 1_000_000
    x, att = o.node2vec_steps(case["t"], case["v"], 2, 0, N, case["p"], case["q"], seed=7)
    counts = [int(np.sum(x == s)) for s in case["support"]]
    assert sum(counts) == N
    probs = [Fraction(p) for p in case["probs"]]
    assert _chi2_p(counts, probs) > P_MIN
    assert np.max(np.abs(np.array(counts) / N - np.array([float(p) for p in probs]))) < 0.01


def _expected_attempts(pg, T, t, v):
    """E[attempts] = 2^32 W_v / sum_x w_vx T_class(x)  (geometric number of draws)."""
    row = pg.rows[v]
    w = [1] * len(row) if pg.cw is None else \
        [pg.cw[v][0]] + [pg.cw[v][i] - pg.cw[v][i - 1] for i in range(1, len(row))]
    acc = 0
    for x, wx in zip(row, w):
        c = 0 if x == t else (1 if pg.member(t, x) else 2)
        acc += wx * T[c]
    return Fraction(2 ** 32 * sum(w), acc)


PQ = [(0.25, 4.0), (4.0, 0.25), (0.5, 2.0), (2.0, 0.5), (1.0, 0.25), (0.25, 1.0), (1.0, 1.0), (3.0, 0.7)]


@pytest.mark.parametrize("p,q", PQ)
@pytest.mark.parametrize("weighted", [False, True])
def test_node2vec_law_on_random_graphs(p, q, weighted):
    """Every (t, v) context of 3 random <= 30-node graphs: the empirical step law
    matches Eq.1 normalised (P:415-426 via P:453-495), and the attempt count
    matches its geometric expectation."""
    T = pyoracle.thresholds(p, q)
    n_ctx = 0
    for gseed in range(3):
        g = tiny_graph(100 + gseed, 12 + 6 * gseed, 0.3, directed=(gseed == 2), weighted=weighted)
        n, off, col, w = g.numpy()
        o = Oracle(n, off, col, w)
        pg = pyoracle.PyGraph(n, off, col, w)
        rng = np.random.default_rng(gseed)
        ctxs = [(t, v) for t in range(n) for v in pg.rows[t] if pg.rows[v]]
        for idx in rng.choice(len(ctxs), size=min(6, len(ctxs)), replace=False):
            t, v = ctxs[idx]
            N = 100_000
            x, att = o.node2vec_steps(t, v, 5, 1000 * idx, N, p, q, seed=gseed + 11)
            law = pyoracle.eq1_law(pg, t, v, p, q)
            support = sorted(law)
            counts = [int(np.sum(x == s)) for s in support]
            assert sum(counts) == N
            assert _chi2_p(counts, [law[s] for s in support]) > P_MIN, (t, v, p, q)
            ea = float(_expected_attempts(pg, T, t, v))
            se = np.sqrt(max(ea * (ea - 1), 1e-12) / N)
            assert abs(att.mean() - ea) < 6 * se + 1e-9
            n_ctx += 1
    assert n_ctx >= 10


@pytest.mark.parametrize("mutation", ["swap-1-q", "drop-return"])
def test_mutants_fail_the_law_test(mutation):
    """Test power: a sampler that swaps the in-N(t) / not-in-N(t) classes, or
    forgets the return class, is rejected by the same chi-square test that the
    correct sampler passes (S:246 example, 20,000 pure-Python draws)."""
    case = LAWS["node2vec"][0]
    n, off, col, w = _graph_from_edges(case["n"], case["edges"], None)
    pg = pyoracle.PyGraph(n, off, col, w)
    T = pyoracle.thresholds(case["p"], case["q"])
    probs = [Fraction(p) for p in case["probs"]]
    N = 20_000

    def counts_for(mut):
        xs = [pg.node2vec_step(T, 9, wid, 2, case["t"], case["v"], mut)[0] for wid in range(N)]
        return [xs.count(s) for s in case["support"]]

    assert _chi2_p(counts_for(None), probs) > P_MIN
    assert _chi2_p(counts_for(mutation), probs) < 1e-12


# --------------------------------------------------------------------------- whole walks
def _path_law(n, p, q, start, L):
    """Path 0-1-...-(n-1), unweighted: first step uniform; interior node coming
    from t returns with q/(p+q) and goes on with p/(p+q) (alpha = 1/p vs 1/q,
    the two neighbours are t and a node at distance 2); endpoints are forced."""
    p, q = Fraction(p), Fraction(q)
    law = {}

    def rec(walk, pr):
        if len(walk) == L:
            law[tuple(walk)] = law.get(tuple(walk), 0) + pr
            return
        v = walk[-1]
        nb = [u for u in (v - 1, v + 1) if 0 <= u < n]
        if len(walk) == 1 or len(nb) == 1:
            for u in nb:
                rec(walk + [u], pr / len(nb))
            return
        t = walk[-2]
        for u in nb:
            rec(walk + [u], pr * (q / (p + q) if u == t else p / (p + q)))
    rec([start], Fraction(1))
    return law


def _star_law(k, p, q, start, L):
    """Star, centre 0, leaves 1..k: at the centre coming from leaf l, back to l
    with q/(q+(k-1)p), each other leaf p/(q+(k-1)p) (leaves are at distance 2
    from each other); leaf -> centre is forced; first step from the centre is uniform."""
    p, q = Fraction(p), Fraction(q)
    law = {}

    def rec(walk, pr):
        if len(walk) == L:
            law[tuple(walk)] = law.get(tuple(walk), 0) + pr
            return
        v = walk[-1]
        if v != 0:
            rec(walk + [0], pr)
            return
        if len(walk) == 1:
            for u in range(1, k + 1):
                rec(walk + [u], pr / k)
            return
        t = walk[-2]
        for u in range(1, k + 1):
            rec(walk + [u], pr * (q / (q + (k - 1) * p) if u == t else p / (q + (k - 1) * p)))
    rec([start], Fraction(1))
    return law


def _triangle_law(p, start, L):
    """Triangle: at v coming from t, back with 1/(1+p), to the third node (a
    neighbour of t) with p/(1+p); q never matters; first step uniform."""
    p = Fraction(p)
    law = {}

    def rec(walk, pr):
        if len(walk) == L:
            law[tuple(walk)] = law.get(tuple(walk), 0) + pr
            return
        v = walk[-1]
        nb = [u for u in range(3) if u != v]
        if len(walk) == 1:
            for u in nb:
                rec(walk + [u], pr / 2)
            return
        t = walk[-2]
        for u in nb:
            rec(walk + [u], pr * (1 / (1 + p) if u == t else p / (1 + p)))
    rec([start], Fraction(1))
    return law


def _csr(n, adj):
    off = np.zeros(n + 1, dtype=np.uint64)
    for v in range(n):
        off[v + 1] = off[v] + len(adj[v])
    col = np.array([u for v in range(n) for u in sorted(adj[v])], dtype=np.uint32)
    return off, col


def _check_walk_law(o, law, start, L, p, q, N, seed):
    out, _ = o.walks(np.full(N, start, dtype=np.uint32), L, mode="node2vec", p=p, q=q, seed=seed)
    keys = sorted(law)
    index = {k: i for i, k in enumerate(keys)}
    counts = np.zeros(len(keys))
    for row in map(tuple, out.tolist()):
        assert row in index, row        # every sampled walk has positive exact probability
        counts[index[row]] += 1
    probs = [law[k] for k in keys]
    assert sum(probs) == 1
    assert _chi2_p(counts, probs) > P_MIN


@pytest.mark.parametrize("p,q", [(0.5, 2.0), (2.0, 0.5), (0.25, 4.0), (1.0, 0.25)])
def test_enumerated_walk_laws_path_star_triangle(p, q):
    N, L = 200_000, 6
    n = 5
    adj = {v: [u for u in (v - 1, v + 1) if 0 <= u < n] for v in range(n)}
    off, col = _csr(n, adj)
    _check_walk_law(Oracle(n, off, col, None), _path_law(n, p, q, 2, L), 2, L, p, q, N, 3)
    k = 4
    adj = {0: list(range(1, k + 1)), **{v: [0] for v in range(1, k + 1)}}
    off, col = _csr(k + 1, adj)
    _check_walk_law(Oracle(k + 1, off, col, None), _star_law(k, p, q, 0, L), 0, L, p, q, N, 4)
    adj = {0: [1, 2], 1: [0, 2], 2: [0, 1]}
    off, col = _csr(3, adj)
    _check_walk_law(Oracle(3, off, col, None), _triangle_law(p, 1, L), 1, L, p, q, N, 5)


def test_stationary_law_of_weighted_first_order_walks():
    """On a connected non-bipartite undirected weighted graph, long first-order
    walks visit v in proportion to its strength s(v) = sum_x w_vx (reversible
    chain with P(v->x) = w_vx / s(v))."""
    g = tiny_graph(77, 16, 0.45, weighted=True, max_w=9)
    n, off, col, w = g.numpy()
    assert np.all(off[1:] > off[:-1])
    o = Oracle(n, off, col, w)
    out, _ = o.walks(np.zeros(400, dtype=np.uint32), 3000, mode="first_order", seed=1)
    visits = np.bincount(out[:, 100:].ravel(), minlength=n).astype(float)
    strength = np.array([int(w[off[v]:off[v + 1]].astype(np.int64).sum()) for v in range(n)], float)
    share, target = visits / visits.sum(), strength / strength.sum()
    assert np.max(np.abs(share - target) / target) < 0.03


# --------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("directed", [False, True])
@pytest.mark.parametrize("mode,p,q", [("first_order", 1, 1), ("node2vec", 0.5, 2.0), ("node2vec", 4.0, 0.25)])
def test_walk_invariants(directed, mode, p, q):
    g = tiny_graph(3, 60, 0.06, directed=directed, weighted=True)
    n, off, col, w = g.numpy()
    o = Oracle(n, off, col, w)
    starts = np.concatenate([np.arange(n), [n, 2 ** 32 - 1]]).astype(np.uint32)
    L = 25
    out, steps = o.walks(starts, L, mode=mode, p=p, q=q, seed=9)
    arcs = {(a, int(c)) for a in range(n) for c in col[off[a]:off[a + 1]]}
    realised = 0
    for i, row in enumerate(out.tolist()):
        if starts[i] >= n:
            assert all(x == pyoracle.PAD for x in row)
            continue
        assert row[0] == starts[i]
        k = next((j for j, x in enumerate(row) if x == pyoracle.PAD), L)
        assert all(x == pyoracle.PAD for x in row[k:])           # PAD only as a suffix
        for a, b in zip(row[:k - 1], row[1:k]):
            assert (a, b) in arcs                                  # every step is an arc
        if k < L:
            assert off[row[k - 1] + 1] == off[row[k - 1]]          # ... and only after a dead end
        realised += k - 1
    assert realised == steps
    out2, _ = o.walks(starts, L, mode=mode, p=p, q=q, seed=9)
    assert np.array_equal(out, out2)


def test_identities_p_q_one_and_unit_weights():
    """node2vec with p = q = 1 is bit-identical to first order (§8(c) c2 + all
    T = 2^32); all-ones weights are bit-identical to unweighted (BOUNDED of the
    same W = deg, upper_bound of i+1 > r gives i = r)."""
    g = tiny_graph(8, 50, 0.1, weighted=False)
    n, off, col, _ = g.numpy()
    starts = np.arange(n, dtype=np.uint32)
    a, _ = Oracle(n, off, col, None).walks(starts, 30, mode="node2vec", p=1.0, q=1.0, seed=3)
    b, _ = Oracle(n, off, col, None).walks(starts, 30, mode="first_order", seed=3)
    c, _ = Oracle(n, off, col, np.ones(len(col), np.uint32)).walks(starts, 30, mode="node2vec",
                                                                    p=2.0, q=0.5, seed=3)
    d, _ = Oracle(n, off, col, None).walks(starts, 30, mode="node2vec", p=2.0, q=0.5, seed=3)
    assert np.array_equal(a, b)
    assert np.array_equal(c, d)


def test_walk_i_alone_equals_row_i():
    g = tiny_graph(21, 40, 0.15, weighted=True)
    n, off, col, w = g.numpy()
    o = Oracle(n, off, col, w)
    starts = np.arange(n, dtype=np.uint32)
    full, _ = o.walks(starts, 20, p=0.5, q=2.0, seed=5, base=100)
    for i in range(0, n, 7):
        one, _ = o.walks(starts[i:i + 1], 20, p=0.5, q=2.0, seed=5, base=100 + i)
        assert np.array_equal(one[0], full[i])

"""Pins of the approximated-walk oracle (SUSS) against what
the paper and SPEC fix (§4.3.3, Fig. 3):

* SUSS "divides the range into k uniformly spaced buckets and then randomly
  samples a value in each bucket" -> k sorted, distinct indices, one uniform
  draw per bucket (structure + per-bucket uniformity);
* "if degree(v) <= d_T the step is exactly the exact-walk step" ->
  bit-identical walks on graphs whose degrees never exceed d_T;
* the step law on the sub-sampled neighbourhood: the exact rules (P:509-511
  steps 1-4, Eq.1) applied to the candidates, averaged over the sub-samples ->
  closed forms (star) and brute-force enumeration of every sub-sample (tiny
  graphs) compared by chi-square with the oracle's samples;
* the pure-Python transliteration agrees with the C oracle bit for bit.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

from oracle import pyoracle
from oracle.oracle import Oracle, suss
from graphgen import tiny_graph

P_MIN = 1e-6


def _chi2_p(counts, probs):
    counts = np.asarray(counts, dtype=np.float64)
    exp = np.asarray([float(p) for p in probs]) * counts.sum()
    return stats.chisquare(counts, exp).pvalue


def _buckets(n, k):
    return [(b * n // k, (b + 1) * n // k) for b in range(k)]


def test_suss_structure_and_paper_example():
    """Fig. 3: d_T = 5 of 15 neighbours -> 5 sorted unique indices,
    one per bucket of width 3; plus random (n, k) with n > k, incl. uneven widths."""
    for wid in range(200):
        idx = suss(42, wid, 1, 15, 5)
        assert len(idx) == 5
        assert all(3 * b <= int(idx[b]) < 3 * b + 3 for b in range(5))
    rng = np.random.default_rng(0)
    for _ in range(300):
        k = int(rng.integers(1, 40))
        n = int(rng.integers(k + 1, 5000))
        idx = [int(v) for v in suss(7, int(rng.integers(0, 2 ** 40)), int(rng.integers(1, 100)), n, k)]
        assert len(idx) == k and all(a < b for a, b in zip(idx, idx[1:]))
        assert all(lo <= c < hi for c, (lo, hi) in zip(idx, _buckets(n, k)))


@pytest.mark.parametrize("n,k", [(100, 10), (23, 5), (7, 3)])
def test_suss_per_bucket_uniformity(n, k):
    """with n=100, k=10 each index is selected with frequency 1/(bucket width)
    = 0.1; in general uniform within its bucket (chi-square per bucket)."""
    counts = np.zeros(n, dtype=np.int64)
    W = 40000
    for wid in range(W):
        counts[np.asarray(suss(3, wid, 5, n, k), dtype=np.int64)] += 1
    for lo, hi in _buckets(n, k):
        c = counts[lo:hi]
        assert c.sum() == W
        assert _chi2_p(c, [Fraction(1, hi - lo)] * (hi - lo)) > P_MIN
    if (n, k) == (100, 10):
        assert np.all(np.abs(counts / W - 0.1) < 0.01)


def test_suss_bucket_pairs_share_a_philox_block_but_differ():
    """Buckets 2j and 2j+1 take the two halves of one Philox block (counter word
    2^31 + j, DESIGN.md f1 reading); the halves differ, and the block differs from
    any attempt's draw (attempt counters stay below 2^31)."""
    from oracle.oracle import draw
    o = draw(11, 5, 3, 0x80000000)
    n, k = 1000, 4
    idx = suss(11, 5, 3, n, k)
    h0 = (o[1] << 32) | o[0]
    h1 = (o[3] << 32) | o[2]
    assert int(idx[0]) == 0 + (h0 * 250 >> 64)
    assert int(idx[1]) == 250 + (h1 * 250 >> 64)
    assert draw(11, 5, 3, 0) != o


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("mode,p,q", [("first_order", 1, 1), ("node2vec", 0.5, 2.0), ("node2vec", 2.0, 0.25)])
def test_identity_when_no_degree_exceeds_threshold(weighted, mode, p, q):
    """degree <= d_T -> the exact step, so whole walks are bit-identical."""
    g = tiny_graph(21, 60, 0.15, weighted=weighted)
    o = Oracle(*g.numpy())
    maxdeg = int(np.max(np.diff(g.off.numpy())))
    starts = np.arange(g.n, dtype=np.uint32)
    exact, es = o.walks(starts, 30, mode=mode, p=p, q=q, seed=9)
    for k in (maxdeg, maxdeg + 1, 10 ** 6):
        approx, as_ = o.walks_approx(starts, 30, k, mode=mode, p=p, q=q, seed=9)
        assert np.array_equal(exact, approx) and es == as_
    approx0, _ = o.walks_approx(starts, 30, 0, mode=mode, p=p, q=q, seed=9)   # k = 0: no threshold
    assert np.array_equal(exact, approx0)
    # a threshold below the maximum degree changes some walks (the rule is live)
    low, _ = o.walks_approx(starts, 30, 2, mode=mode, p=p, q=q, seed=9)
    assert not np.array_equal(exact, low)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("weighted,directed", [(False, False), (True, False), (True, True)])
def test_python_transliteration_matches_c(seed, weighted, directed):
    g = tiny_graph(300 + seed, 40, 0.3, weighted=weighted, directed=directed, self_loops=directed)
    n, off, col, w = g.numpy()
    o = Oracle(n, off, col, w)
    pg = pyoracle.PyGraph(n, off, col, w)
    starts = np.concatenate([np.arange(n), [n + 2]]).astype(np.uint32)
    for k in (1, 3, 7):
        for mode, p, q in [("first_order", 1, 1), ("node2vec", 0.5, 2.0), ("node2vec", 4.0, 0.25)]:
            got, steps = o.walks_approx(starts, 12, k, mode=mode, p=p, q=q, seed=seed, base=77)
            tot = 0
            for i, st in enumerate(starts):
                row, s_ = pg.walk_approx(int(st), 77 + i, 12, k, mode=mode, p=p, q=q, seed=seed)
                assert list(got[i]) == row, (k, mode, i)
                tot += s_
            assert tot == steps


def _star(n_leaves, weights=None):
    """Undirected star, centre 0, leaves 1..n."""
    arcs = [(0, j) for j in range(1, n_leaves + 1)] + [(j, 0) for j in range(1, n_leaves + 1)]
    arcs.sort()
    off = np.zeros(n_leaves + 2, dtype=np.uint64)
    for a, _ in arcs:
        off[a + 1] += 1
    off = np.cumsum(off).astype(np.uint64)
    col = np.array([b for _, b in arcs], dtype=np.uint32)
    w = None
    if weights is not None:
        w = np.array([weights[b - 1] if a == 0 else weights[a - 1] for a, b in arcs], dtype=np.uint32)
    return n_leaves + 1, off, col, w


@pytest.mark.parametrize("n,k", [(12, 5), (10, 4)])
def test_first_order_marginal_law_on_a_star(n, k):
    """Unweighted first-order step from the centre of a star with n > k leaves:
    bucket b is chosen with probability 1/k and leaf j of bucket b (width w_b) is
    its candidate with probability 1/w_b, so P(leaf j) = 1 / (k w_b(j)).  With
    uneven buckets this is NOT 1/n — the approximation the paper accepts."""
    g = Oracle(*_star(n))
    W = 200000
    starts = np.zeros(W, dtype=np.uint32)
    rows, _ = g.walks_approx(starts, 2, k, mode="first_order", seed=13)
    counts = np.bincount(rows[:, 1].astype(np.int64), minlength=n + 1)[1:]
    probs = []
    for lo, hi in _buckets(n, k):
        probs += [Fraction(1, k * (hi - lo))] * (hi - lo)
    assert sum(probs) == 1
    assert _chi2_p(counts, probs) > P_MIN


def _enumerated_law(pg, t, v, k, p, q):
    """Exact law of one approximated node2vec step at v (coming from t): the
    average over every equally likely sub-sample (one index per bucket) of the
    Eq.1 law restricted to the candidates (P:415-426 on the Fig. 3b candidates)."""
    row = pg.rows[v]
    n = len(row)
    if pg.cw is None:
        w = [1] * n
    else:
        c = pg.cw[v]
        w = [c[0]] + [c[i] - c[i - 1] for i in range(1, n)]
    p, q = Fraction(p), Fraction(q)
    law = {x: Fraction(0) for x in row}
    subs = list(itertools.product(*[range(lo, hi) for lo, hi in _buckets(n, k)]))
    for cand in subs:
        pis = []
        for j in cand:
            x = row[j]
            alpha = 1 / p if x == t else (Fraction(1) if pg.member(t, x) else 1 / q)
            pis.append(alpha * w[j])
        tot = sum(pis)
        for j, pi in zip(cand, pis):
            law[row[j]] += pi / tot / len(subs)
    return law


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("p,q,k", [(0.5, 2.0, 2), (2.0, 0.25, 3), (1.0, 1.0, 2)])
def test_node2vec_marginal_law_by_enumeration(weighted, p, q, k):
    """Graph: t = 0 with the single neighbour v = 1 (so every walk from t steps to v);
    v has 6 neighbours (t, two of t's other... see edges), k < 6 -> SUSS at v.
    The oracle's row[2] frequencies match the enumerated law (chi-square)."""
    # undirected edges: 0-1, 1-2, 1-3, 1-4, 1-5, 1-6, 2-3 ; plus 0-... none (t = 0 has only v)
    # to make "x in N(t)" non-trivial give t a second neighbour 3 and start walks at 0
    # with the first step forced by weights: 0's row {1, 3} with weight(0,3) tiny.
    edges = [(0, 1), (0, 3), (1, 2), (1, 3), (1, 4), (1, 5), (1, 6), (2, 3)]
    wts = {(0, 1): 10 ** 6, (0, 3): 1, (1, 2): 3, (1, 3): 1, (1, 4): 5, (1, 5): 2, (1, 6): 4, (2, 3): 7}
    arcs = {}
    for (a, b) in edges:
        arcs[(a, b)] = wts[(a, b)]
        arcs[(b, a)] = wts[(a, b)]
    keys = sorted(arcs)
    nn = 7
    off = np.zeros(nn + 1, dtype=np.uint64)
    for a, _ in keys:
        off[a + 1] += 1
    off = np.cumsum(off).astype(np.uint64)
    col = np.array([b for _, b in keys], dtype=np.uint32)
    w = np.array([arcs[kk] for kk in keys], dtype=np.uint32)
    if not weighted:
        # unweighted: the first step from 0 is uniform over {1, 3}; keep only walks via 1
        w = None
    g = Oracle(nn, off, col, w)
    pg = pyoracle.PyGraph(nn, off, col, w)
    law = _enumerated_law(pg, 0, 1, k, p, q)
    W = 120000
    rows, _ = g.walks_approx(np.zeros(W, dtype=np.uint32), 3, k, mode="node2vec", p=p, q=q, seed=5)
    via_v = rows[:, 1] == 1
    xs = rows[via_v, 2].astype(np.int64)
    assert len(xs) > 50000
    support = sorted(law)
    counts = [int(np.sum(xs == x)) for x in support]
    assert sum(counts) == len(xs)
    assert _chi2_p(counts, [law[x] for x in support]) > P_MIN
    # power: the exact (non-sub-sampled) Eq.1 law differs and is rejected when k is small
    exact = pyoracle.eq1_law(pg, 0, 1, p, q)
    if any(abs(float(exact[x] - law[x])) > 0.02 for x in support):
        assert _chi2_p(counts, [exact[x] for x in support]) < 1e-3

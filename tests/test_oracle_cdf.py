"""Pins of the paper's CDF node2vec sampler in the oracle (
P:507-511 §4.3.2 steps 1-4), against what the paper and the mathematics fix:

* the step law is Eq.1: P(x) = alpha_pq(t,x) w_vx / sum — the SPEC
  worked examples [1/7, 2/7, 4/7] and its weighted variant, and the
  exact law of every context of random tiny graphs (chi-square);
* one draw per step: the sampled index is the exact inverse CDF of the draw
  (brute force with Python big integers over many draws);
* p = q = 1 reduces to the first-order walk bit for bit (a proof in DESIGN.md
  §7c; a mistaken scaling of r or of the running sum breaks it);
* the pure-Python transliteration equals the C oracle bit for bit;
* power: mutants (swapped 1/q classes, dropped return class) fail the same tests.
"""
import numpy as np
import pytest
from fractions import Fraction
from scipy import stats

from oracle import pyoracle
from oracle.oracle import Oracle, draw
from graphgen import tiny_graph

P_MIN = 1e-6


def _chi2_p(counts, probs):
    counts = np.asarray(counts, dtype=np.float64)
    exp = np.asarray([float(p) for p in probs]) * counts.sum()
    return stats.chisquare(counts, exp).pvalue


def _graph(n, edges, w=None):
    arcs = {}
    for k, (a, b) in enumerate(edges):
        ww = 1 if w is None else w[k]
        arcs[(a, b)] = ww
        arcs[(b, a)] = ww
    keys = sorted(arcs)
    off = np.zeros(n + 1, dtype=np.uint64)
    for a, _ in keys:
        off[a + 1] += 1
    off = np.cumsum(off).astype(np.uint64)
    col = np.array([b for _, b in keys], dtype=np.uint32)
    wt = None if w is None else np.array([arcs[k] for k in keys], dtype=np.uint32)
    return n, off, col, wt


SPEC_EDGES = [(0, 1), (1, 2), (1, 3), (0, 2)]   # t = 0, v = 1, N(1) = {0, 2, 3}, N(0) = {1, 2}


@pytest.mark.parametrize("weights,expect", [
    (None, [Fraction(1, 7), Fraction(2, 7), Fraction(4, 7)]),          # S:246, p = 2, q = 0.5
    ([1, 3, 5, 1], [Fraction(1, 27), Fraction(6, 27), Fraction(20, 27)]),
])
def test_spec_worked_example(weights, expect):
    g = Oracle(*_graph(4, SPEC_EDGES, weights))
    xs = g.cdf_steps(0, 1, 2, 0, 200000, p=2.0, q=0.5, seed=7)
    counts = [int(np.sum(xs == x)) for x in (0, 2, 3)]
    assert sum(counts) == len(xs)
    assert _chi2_p(counts, expect) > P_MIN


@pytest.mark.parametrize("seed,weighted,directed", [(1, False, False), (2, True, False), (3, True, True)])
@pytest.mark.parametrize("p,q", [(0.5, 2.0), (4.0, 0.25), (2.0, 1.0)])
def test_eq1_law_on_random_graph_contexts(seed, weighted, directed, p, q):
    g = tiny_graph(700 + seed, 24, 0.3, weighted=weighted, directed=directed, self_loops=directed)
    n, off, col, w = g.numpy()
    o = Oracle(n, off, col, w)
    pg = pyoracle.PyGraph(n, off, col, w)
    rng = np.random.default_rng(seed)
    done = 0
    for _ in range(40):
        t = int(rng.integers(0, n))
        if not pg.rows[t]:
            continue
        v = pg.rows[t][int(rng.integers(0, len(pg.rows[t])))]
        if len(pg.rows[v]) < 2:
            continue
        law = pyoracle.eq1_law(pg, t, v, p, q)
        xs = o.cdf_steps(t, v, 3, 1000 * done, 60000, p=p, q=q, seed=seed)
        support = sorted(law)
        counts = [int(np.sum(xs == x)) for x in support]
        assert sum(counts) == len(xs)
        assert _chi2_p(counts, [law[x] for x in support]) > P_MIN
        done += 1
        if done == 4:
            break
    assert done == 4


def test_inverse_cdf_brute_force():
    """The chosen index is the first i with cum_i > floor(x64 * S / 2^64), S = sum of
    w * T_class — recomputed with Python integers for 2000 draws on a weighted row."""
    n, off, col, w = _graph(6, [(0, 1), (1, 2), (1, 3), (1, 4), (1, 5), (0, 2), (2, 3)], [7, 1, 900, 3, 40, 2, 5])
    o = Oracle(n, off, col, w)
    pg = pyoracle.PyGraph(n, off, col, w)
    T = pyoracle.thresholds(0.3, 3.0)
    xs = o.cdf_steps(0, 1, 4, 0, 2000, p=0.3, q=3.0, seed=99)
    row = pg.rows[1]
    c = pg.cw[1]
    ws = [c[i] - (c[i - 1] if i else 0) for i in range(len(c))]
    pis = [wx * (T[0] if x == 0 else (T[1] if pg.member(0, x) else T[2])) for x, wx in zip(row, ws)]
    S = sum(pis)
    for k in range(2000):
        d = draw(99, k, 4, 0)
        r = ((d[1] << 32 | d[0]) * S) >> 64
        acc, pick = 0, None
        for x, pi in zip(row, pis):
            acc += pi
            if acc > r:
                pick = x
                break
        assert int(xs[k]) == pick


@pytest.mark.parametrize("weighted", [False, True])
def test_p_q_one_is_first_order(weighted):
    g = tiny_graph(31, 50, 0.2, weighted=weighted)
    o = Oracle(*g.numpy())
    starts = np.arange(g.n, dtype=np.uint32)
    a, sa = o.walks_cdf(starts, 40, p=1.0, q=1.0, seed=5)
    b, sb = o.walks(starts, 40, mode="first_order", seed=5)
    assert np.array_equal(a, b) and sa == sb


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("weighted,directed", [(False, False), (True, False), (True, True)])
def test_python_transliteration_matches_c(seed, weighted, directed):
    g = tiny_graph(900 + seed, 30, 0.25, weighted=weighted, directed=directed, self_loops=directed)
    n, off, col, w = g.numpy()
    o = Oracle(n, off, col, w)
    pg = pyoracle.PyGraph(n, off, col, w)
    starts = np.concatenate([np.arange(n), [n + 1]]).astype(np.uint32)
    for p, q in [(0.5, 2.0), (4.0, 0.25), (1.0, 3.0)]:
        got, steps = o.walks_cdf(starts, 14, p=p, q=q, seed=seed, base=41)
        tot = 0
        for i, st in enumerate(starts):
            row, s_ = pg.walk_cdf(int(st), 41 + i, 14, p=p, q=q, seed=seed)
            assert list(got[i]) == row
            tot += s_
        assert tot == steps


def test_mutants_fail_the_law():
    """Test power: a CDF step that swaps the 1 / q classes, or treats the return
    like any other node, is rejected by the SPEC example's chi-square."""
    n, off, col, _ = _graph(4, SPEC_EDGES)
    pg = pyoracle.PyGraph(n, off, col)
    T = pyoracle.thresholds(2.0, 0.5)
    expect = [Fraction(1, 7), Fraction(2, 7), Fraction(4, 7)]

    def mutant_step(kind, wid):
        row = pg.rows[1]
        pis = []
        for x in row:
            if x == 0 and kind != "drop-return":
                tc = T[0]
            elif pg.member(0, x):
                tc = T[2] if kind == "swap-1-q" else T[1]
            else:
                tc = T[1] if kind == "swap-1-q" else T[2]
            pis.append(tc)
        d = draw(7, wid, 2, 0)
        r = ((d[1] << 32 | d[0]) * sum(pis)) >> 64
        acc = 0
        for x, pi in zip(row, pis):
            acc += pi
            if acc > r:
                return x

    for kind in ("swap-1-q", "drop-return"):
        xs = np.array([mutant_step(kind, k) for k in range(20000)])
        counts = [int(np.sum(xs == x)) for x in (0, 2, 3)]
        assert _chi2_p(counts, expect) < 1e-6, kind

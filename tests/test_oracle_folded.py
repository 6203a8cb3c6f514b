"""Pins of the outlier-folded rejection rule in the oracle (SURVEY §8(f) row f2,
"outlier-folded proposals"):

* same law as the default rule — Eq.1: the SPEC worked examples and
  the exact law of random contexts (chi-square), including return-heavy
  settings (p < min(1, q)) where folding is active;
* bit-identical to the default rule whenever p >= min(1, q) (folding inactive);
* fewer attempts than the default rule when p < min(1, q), matching the
  geometric expectation M / sum_x w_vx T_c(x) * 2^32 / ... (exact formula below);
* the pure-Python transliteration equals the C oracle bit for bit;
* power: a mutant that forgets the return's excess mass (N) is rejected.
"""
from fractions import Fraction

import numpy as np
import pytest
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


SPEC_EDGES = [(0, 1), (1, 2), (1, 3), (0, 2)]


@pytest.mark.parametrize("p,q", [(2.0, 0.5), (0.25, 4.0), (0.5, 2.0)])
@pytest.mark.parametrize("weights", [None, [1, 3, 5, 1]])
def test_spec_example_law(p, q, weights):
    g = Oracle(*_graph(4, SPEC_EDGES, weights))
    pg = pyoracle.PyGraph(*_graph(4, SPEC_EDGES, weights))
    law = pyoracle.eq1_law(pg, 0, 1, p, q)
    xs, _ = g.folded_steps(0, 1, 2, 0, 200000, p=p, q=q, seed=7)
    support = sorted(law)
    counts = [int(np.sum(xs == x)) for x in support]
    assert _chi2_p(counts, [law[x] for x in support]) > P_MIN


@pytest.mark.parametrize("seed,weighted,directed", [(1, False, False), (2, True, False), (3, True, True)])
@pytest.mark.parametrize("p,q", [(0.25, 4.0), (0.5, 2.0), (0.3, 1.0)])
def test_eq1_law_on_random_contexts(seed, weighted, directed, p, q):
    g = tiny_graph(800 + seed, 24, 0.3, weighted=weighted, directed=directed, self_loops=directed)
    n, off, col, w = g.numpy()
    o = Oracle(n, off, col, w)
    pg = pyoracle.PyGraph(n, off, col, w)
    rng = np.random.default_rng(seed)
    done = 0
    for _ in range(60):
        t = int(rng.integers(0, n))
        if not pg.rows[t]:
            continue
        v = pg.rows[t][int(rng.integers(0, len(pg.rows[t])))]
        if len(pg.rows[v]) < 2:
            continue
        law = pyoracle.eq1_law(pg, t, v, p, q)
        xs, _ = o.folded_steps(t, v, 3, 1000 * done, 60000, p=p, q=q, seed=seed)
        support = sorted(law)
        counts = [int(np.sum(xs == x)) for x in support]
        assert sum(counts) == len(xs)
        assert _chi2_p(counts, [law[x] for x in support]) > P_MIN
        done += 1
        if done == 4:
            break
    assert done == 4


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("p,q", [(2.0, 0.5), (1.0, 0.25), (4.0, 1.0), (1.0, 1.0), (1.0, 3.0)])
def test_identical_to_default_rule_when_not_return_heavy(weighted, p, q):
    """p >= min(1, q): E = 2^32, no excess, A = T — the default rule, draw for draw."""
    g = tiny_graph(41, 60, 0.15, weighted=weighted)
    o = Oracle(*g.numpy())
    starts = np.arange(g.n, dtype=np.uint32)
    a, sa = o.walks_folded(starts, 40, p=p, q=q, seed=3)
    b, sb = o.walks(starts, 40, mode="node2vec", p=p, q=q, seed=3)
    assert np.array_equal(a, b) and sa == sb


@pytest.mark.parametrize("p,q", [(0.25, 4.0), (0.5, 2.0)])
def test_fewer_attempts_and_their_expectation(p, q):
    """Return-heavy settings: mean attempts per step = M / sum_x w_vx min(T_c,E) + N ... i.e.
    E[attempts] = M / (M_accepted) with M = W E + N and M_accepted = N + sum_x w_vx A_c E / 2^32;
    compared with the oracle's counts, and smaller than the default rule's."""
    n, off, col, w = _graph(6, [(0, 1), (1, 2), (1, 3), (1, 4), (1, 5), (0, 2)], [5, 1, 2, 3, 4, 1])
    o = Oracle(n, off, col, w)
    pg = pyoracle.PyGraph(n, off, col, w)
    T = pyoracle.thresholds(p, q)
    E = max(T[1], T[2])
    X = T[0] - E if T[0] > E else 0
    A = [-(-(min(tc, E) << 32) // E) for tc in T]
    row = pg.rows[1]
    c = pg.cw[1]
    ws = [c[i] - (c[i - 1] if i else 0) for i in range(len(c))]
    W = c[-1]
    wt = ws[row.index(0)]
    N = wt * X
    M = W * E + N
    # per attempt: P(outlier) = ceil(N 2^32 / M) / 2^32 (o3 * M < N 2^32), else a proposal x
    # (probability w_x / W) accepted with probability A_class / 2^32
    p_out = Fraction(-(-(N << 32) // M), 1 << 32) if N else Fraction(0)
    p_acc_reg = sum(Fraction(wx, W) * Fraction(A[0] if x == 0 else (A[1] if pg.member(0, x) else A[2]), 1 << 32)
                    for x, wx in zip(row, ws))
    p_step = p_out + (1 - p_out) * p_acc_reg
    _, att = o.folded_steps(0, 1, 2, 0, 200000, p=p, q=q, seed=11)
    _, att_d = o.node2vec_steps(0, 1, 2, 0, 200000, p=p, q=q, seed=11)
    mean = float(np.mean(att))
    expect = float(1 / p_step)
    sd = float(np.sqrt(float((1 - p_step) / p_step ** 2)) / np.sqrt(len(att)))
    assert abs(mean - expect) < 6 * sd
    assert mean < float(np.mean(att_d))


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("weighted,directed", [(False, False), (True, False), (True, True)])
def test_python_transliteration_matches_c(seed, weighted, directed):
    g = tiny_graph(950 + seed, 30, 0.25, weighted=weighted, directed=directed, self_loops=directed)
    n, off, col, w = g.numpy()
    o = Oracle(n, off, col, w)
    pg = pyoracle.PyGraph(n, off, col, w)
    starts = np.concatenate([np.arange(n), [n + 1]]).astype(np.uint32)
    for p, q in [(0.25, 4.0), (0.5, 2.0), (2.0, 0.5)]:
        got, steps = o.walks_folded(starts, 14, p=p, q=q, seed=seed, base=19)
        tot = 0
        for i, st in enumerate(starts):
            row, s_ = pg.walk_folded(int(st), 19 + i, 14, p=p, q=q, seed=seed)
            assert list(got[i]) == row
            tot += s_
        assert tot == steps


def test_mutant_without_excess_mass_fails():
    """Dropping the return's excess N (the outlier branch) under-samples the return."""
    n, off, col, _ = _graph(4, SPEC_EDGES)
    pg = pyoracle.PyGraph(n, off, col)
    p, q = 0.25, 4.0
    law = pyoracle.eq1_law(pg, 0, 1, p, q)
    T = pyoracle.thresholds(p, q)
    E = max(T[1], T[2])
    A = [-(-(min(tc, E) << 32) // E) for tc in T]
    xs = []
    for k in range(40000):
        a = 0
        while True:
            o = draw(7, k, 2, a)
            a += 1
            x = pg.propose(1, (o[1] << 32) | o[0])
            thr = A[0] if x == 0 else (A[1] if pg.member(0, x) else A[2])
            if o[2] < thr:
                xs.append(x)
                break
    xs = np.array(xs)
    support = sorted(law)
    counts = [int(np.sum(xs == x)) for x in support]
    assert _chi2_p(counts, [law[x] for x in support]) < 1e-6

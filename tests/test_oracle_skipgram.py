"""Pins of the SkipGram consumer in the oracle,
against what the paper and the mathematics fix:

* rank (P:405's Elias-Fano rank): for EVERY arc index of graphs with isolated
  nodes, the node whose row holds it — brute force from the arc-source array;
* scale-free negatives ("outbound ... node degrees scale-free
  distribution"): chi-square of the negatives against deg(v) / m; isolated
  nodes never drawn; power: a uniform-over-nodes sampler is rejected;
* pairs (the sliding window, the context of a central node): the
  number of pairs of a row with l live entries in closed form, the pair multiset
  symmetric, every pair at distance <= w inside one walk, PAD-suffix rows;
* slots are a function of the global walk id: a shard (base = its first wid)
  reproduces its slice of the whole matrix's output bit for bit;
* the pure-Python transliteration equals the C oracle bit for bit.
"""
import numpy as np
import pytest
from scipy import stats

from graphgen import tiny_graph
from oracle import pyoracle
from oracle.oracle import Oracle

PAD = 0xFFFFFFFF


def _graph_with_isolated(seed, n=40, dens=0.12, directed=False):
    """tiny_graph on n nodes spread monotonically over n + n//3 ids: the other ids
    (some adjacent, possibly the first and last) are isolated rows."""
    g = tiny_graph(seed, n, dens, directed=directed, weighted=False, self_loops=False)
    n0, off0, col0, _ = g.numpy()
    rng = np.random.default_rng(seed)
    N = n0 + n0 // 3
    ids = np.sort(rng.choice(N, n0, replace=False))      # monotone: rows stay sorted
    deg = np.zeros(N, dtype=np.int64)
    deg[ids] = np.diff(off0.astype(np.int64))
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    col = ids[col0.astype(np.int64)].astype(np.uint32)
    return N, off, col, None


@pytest.mark.parametrize("seed,directed", [(1, False), (2, True), (3, False)])
def test_rank_every_arc_index(seed, directed):
    n, off, col, w = _graph_with_isolated(300 + seed, directed=directed)
    deg = np.diff(off.astype(np.int64))
    src = np.repeat(np.arange(n), deg)          # the source node of every arc, in arc order
    assert (deg == 0).any()                      # the case rank must skip
    o = Oracle(n, off, col, w)
    for e in range(int(off[-1])):
        assert o.rank(e) == src[e]


def test_rank_runs_of_empty_rows():
    off = np.array([0, 0, 0, 3, 3, 5, 5, 5, 6], dtype=np.uint64)   # rows 0,1 / 3 / 5,6 empty
    o = Oracle(8, off, np.zeros(6, dtype=np.uint32))
    assert [o.rank(e) for e in range(6)] == [2, 2, 2, 4, 4, 7]


def _live_walks(seed, o, n, W, L):
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, n + 2, W).astype(np.uint32)     # a few bad starts: all-PAD rows
    walks, _ = o.walks(starts, L, mode="node2vec", p=0.5, q=2.0, seed=seed)
    return walks


@pytest.mark.parametrize("window", [1, 3, 5])
def test_pairs_closed_form_and_symmetry(window):
    n, off, col, w = _graph_with_isolated(11)
    o = Oracle(n, off, col, w)
    L = 12
    walks = _live_walks(5, o, n, 200, L)
    c, x, _ = o.skipgram(walks, window, 0)
    S = walks.shape[0] * L * 2 * window
    assert c.shape == (S,)
    live = (walks != PAD).sum(axis=1)
    assert np.all(np.cumsum(walks == PAD, axis=1)[walks != PAD] == 0)     # PAD is a suffix
    # a row with l live entries: sum_i min(w, i) + min(w, l-1-i) pairs
    expect = sum(sum(min(window, i) + min(window, ll - 1 - i) for i in range(ll)) for ll in live)
    valid = c != PAD
    assert np.array_equal(valid, x != PAD) and valid.sum() == expect
    # symmetric multiset: (a, b) occurs as often as (b, a)
    pairs = np.stack([c[valid], x[valid]], 1).astype(np.int64)
    fw = {tuple(r) for r in pairs.tolist()}
    cnt = {}
    for a, b in pairs.tolist():
        cnt[(a, b)] = cnt.get((a, b), 0) + 1
    assert all(cnt[(a, b)] == cnt.get((b, a), 0) for a, b in fw)
    # each slot: the context is the entry at offset j of the same row
    slots = np.nonzero(valid)[0]
    r = slots // (L * 2 * window)
    i = (slots // (2 * window)) % L
    oo = slots % (2 * window)
    j = np.where(oo < window, oo - window, oo - window + 1)
    assert np.all(np.abs(j) <= window) and np.all(j != 0)
    assert np.array_equal(walks[r, i], c[slots]) and np.array_equal(walks[r, i + j], x[slots])


@pytest.mark.parametrize("directed", [False, True])
def test_negatives_follow_out_degree(directed):
    n, off, col, w = _graph_with_isolated(21, n=30, dens=0.15, directed=directed)
    o = Oracle(n, off, col, w)
    deg = np.diff(off.astype(np.int64))
    walks = np.tile(np.array([[int(np.argmax(deg)), int(col[off[np.argmax(deg)]])]], dtype=np.uint32), (4000, 1))
    _, _, ng = o.skipgram(walks, 1, 8, seed=3)
    neg = ng[ng != PAD]
    assert len(neg) == 4000 * 2 * 8
    counts = np.bincount(neg.astype(np.int64), minlength=n)
    assert np.all(counts[deg == 0] == 0)
    sup = deg > 0
    p = stats.chisquare(counts[sup], deg[sup] / deg.sum() * len(neg)).pvalue
    assert p > 1e-6
    # power: a negative sampler uniform over the nodes of positive degree is rejected
    rng = np.random.default_rng(0)
    unif = rng.choice(np.nonzero(sup)[0], len(neg))
    cu = np.bincount(unif, minlength=n)
    assert stats.chisquare(cu[sup], deg[sup] / deg.sum() * len(neg)).pvalue < 1e-6


def test_shard_slices_and_python_transliteration():
    n, off, col, w = _graph_with_isolated(31, n=25, dens=0.2)
    o = Oracle(n, off, col, w)
    L, win, K = 7, 2, 3
    walks = _live_walks(9, o, n, 30, L)
    c, x, ng = o.skipgram(walks, win, K, seed=77)
    per = L * 2 * win
    for a, b in ((0, 11), (11, 12), (12, 30)):
        cs, xs, ns = o.skipgram(walks[a:b], win, K, seed=77, base=a)
        assert np.array_equal(cs, c[a * per:b * per]) and np.array_equal(xs, x[a * per:b * per])
        assert np.array_equal(ns, ng[a * per:b * per])
    pg = pyoracle.PyGraph(n, off, col)
    pc, px, pn = pyoracle.skipgram(pg, walks.tolist(), win, K, seed=77)
    assert pc == c.tolist() and px == x.tolist() and pn == ng.tolist()


def test_no_arcs_means_no_pairs():
    o = Oracle(3, np.zeros(4, dtype=np.uint64), np.zeros(0, dtype=np.uint32))
    walks = np.array([[0, PAD, PAD], [2, PAD, PAD]], dtype=np.uint32)
    c, x, ng = o.skipgram(walks, 2, 2)
    assert np.all(c == PAD) and np.all(x == PAD) and np.all(ng == PAD)

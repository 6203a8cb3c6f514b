"""Pins of the oracle's arithmetic against things other than itself.

* Philox4x32-10 vs the CUDA toolkit's independent curand_Philox4x32_10 (host).
* Known-answer draws / walks (tests/golden/kat_*.json).
* BOUNDED vs the exact preimage law of floor(x W / 2^64).
* upper_bound vs linear scan, exhaustively on small rows.
* thresholds vs exact rationals (closed forms of §8(c) c9).
* prefix sums vs numpy cumsum.
* C oracle vs the independent pure-Python transliteration, bit for bit.
"""
import json
import math
import os
import subprocess
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st, HealthCheck

import oracle
from oracle import pyoracle
from oracle.oracle import Oracle, _LIB
from graphgen import tiny_graph

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _hex(v):
    return int(v, 16) if isinstance(v, str) else int(v)


# --------------------------------------------------------------------------- Philox
def test_philox_matches_curand_toolkit_implementation(tmp_path):
    """oracle Philox == curand_Philox4x32_10 on 10^6 random (ctr, key) + edge patterns."""
    exe = tmp_path / "pin"
    src = os.path.join(HERE, "pins", "curand_philox_pin.cu")
    libdir = os.path.dirname(_LIB)
    subprocess.check_call(["nvcc", "-O2", "-Wno-deprecated-gpu-targets", "-o", str(exe), src,
                           f"-L{libdir}", "-loracle", f"-Xlinker", f"-rpath={libdir}"],
                          cwd=str(tmp_path))
    out = subprocess.run([str(exe), "1000000", "12345"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches=0" in out.stdout


def test_philox_python_transliteration_agrees():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        c = [int(v) for v in rng.integers(0, 2 ** 32, 4, dtype=np.uint64)]
        k = [int(v) for v in rng.integers(0, 2 ** 32, 2, dtype=np.uint64)]
        assert oracle.philox4x32_10(c, k) == pyoracle.philox4x32_10(c, k)


def test_known_answer_draws():
    kat = json.load(open(os.path.join(GOLD, "kat_draws.json")))
    for d in kat["draws"]:
        seed, wid = _hex(d["seed"]), _hex(d["wid"])
        o = oracle.draw(seed, wid, d["s"], d["a"])
        assert o == tuple(_hex(v) for v in d["o"])
        assert pyoracle.draw(seed, wid, d["s"], d["a"]) == o
        x64 = (o[1] << 32) | o[0]
        assert x64 == _hex(d["x64"]) and o[2] == _hex(d["u"])
        assert oracle.bounded(x64, 3) == d["bounded3"]
        assert oracle.bounded(x64, 100) == d["bounded100"]


def test_known_answer_walks():
    kat = json.load(open(os.path.join(GOLD, "kat_walks.json")))
    for wk in kat["walks"]:
        g = kat["graphs"][wk["graph"]]
        o = Oracle(g["n"], np.array(g["off"]), np.array(g["col"]), None)
        out, steps, att = o.walks([wk["start"]], wk["L"], mode=wk["mode"], p=wk["p"], q=wk["q"],
                                  seed=42, base=wk["wid"], with_attempts=True)
        assert out[0].tolist() == wk["row"], wk
        if "attempts" in wk:
            assert att == wk["attempts"]
        pg = pyoracle.PyGraph(g["n"], g["off"], g["col"])
        row, _ = pg.walk(wk["start"], wk["wid"], wk["L"], wk["mode"], wk["p"], wk["q"], 42)
        assert row == wk["row"]


def test_attempt_counter_mutation_is_caught_by_kat():
    """Shifting the attempt counter keeps the law but breaks the convention: the
    bit-exact KAT (not the chi-square tests) is what catches it."""
    kat = json.load(open(os.path.join(GOLD, "kat_walks.json")))
    wk = kat["walks"][1]
    g = kat["graphs"][wk["graph"]]
    pg = pyoracle.PyGraph(g["n"], g["off"], g["col"])
    row, _ = pg.walk(wk["start"], wk["wid"], wk["L"], wk["mode"], wk["p"], wk["q"], 42,
                     mutation="attempt+1")
    assert row != wk["row"]


# --------------------------------------------------------------------------- BOUNDED
@pytest.mark.parametrize("W", [1, 2, 3, 7, 100, 1000, 2 ** 31 + 11, 2 ** 40 + 3, 2 ** 64 - 1])
def test_bounded_special_values_and_preimage_law(W):
    assert oracle.bounded(0, W) == 0
    assert oracle.bounded(2 ** 64 - 1, W) == W - 1
    # floor(x W / 2^64) = r  <=>  ceil(r 2^64 / W) <= x < ceil((r+1) 2^64 / W):
    # each outcome r has exactly ceil((r+1) 2^64/W) - ceil(r 2^64/W) preimages.
    rng = np.random.default_rng(W % 1000)
    for r in set([0, W - 1] + [int(v) for v in rng.integers(0, min(W, 2 ** 62), 20)]):
        lo = -((-r * 2 ** 64) // W)
        hi = -((-(r + 1) * 2 ** 64) // W)
        assert hi > lo
        assert oracle.bounded(lo, W) == r
        assert oracle.bounded(hi - 1, W) == r
        if lo > 0:
            assert oracle.bounded(lo - 1, W) == r - 1
        if hi < 2 ** 64:
            assert oracle.bounded(hi, W) == r + 1


@settings(max_examples=300, deadline=None)
@given(st.integers(0, 2 ** 64 - 1), st.integers(1, 2 ** 64 - 1))
def test_bounded_range_and_monotone(x, W):
    r = oracle.bounded(x, W)
    assert 0 <= r < W
    assert r * 2 ** 64 <= x * W < (r + 1) * 2 ** 64


# --------------------------------------------------------------------------- search
def test_upper_bound_exhaustive_vs_linear_scan():
    rng = np.random.default_rng(1)
    for d in [1, 2, 3, 5, 8, 17, 64, 129]:
        for _ in range(5):
            w = rng.integers(1, 6, d).astype(np.uint64)
            cw = np.cumsum(w).astype(np.uint64)
            for r in range(int(cw[-1])):
                lin = next(i for i in range(d) if int(cw[i]) > r)
                assert oracle.upper_bound(cw, r) == lin


# --------------------------------------------------------------------------- thresholds
def test_thresholds_closed_forms_for_every_config():
    """§8(c) c9: the BASELINE configs' ratios are powers of two, so T is exact."""
    assert oracle.thresholds(0.5, 2.0) == (2 ** 32, 2 ** 31, 2 ** 30)   # cfg2
    assert oracle.thresholds(1.0, 0.25) == (2 ** 30, 2 ** 30, 2 ** 32)  # cfg3
    assert oracle.thresholds(2.0, 0.5) == (2 ** 30, 2 ** 31, 2 ** 32)   # cfg4
    assert oracle.thresholds(0.25, 4.0) == (2 ** 32, 2 ** 30, 2 ** 28)  # cfg5
    assert oracle.thresholds(1.0, 1.0) == (2 ** 32, 2 ** 32, 2 ** 32)


@pytest.mark.parametrize("p,q", [(0, 1), (-1, 1), (1, 0), (float("nan"), 1), (1, float("inf")),
                                 (2.0 ** 25, 1.0), (1.0, 2.0 ** -24.5), (2.0 ** 12, 2.0 ** -12.5)])
def test_thresholds_reject(p, q):
    assert oracle.thresholds(p, q) is None
    assert pyoracle.thresholds(p, q) is None


@settings(max_examples=400, deadline=None)
@given(st.floats(2 ** -12, 2 ** 12), st.floats(2 ** -12, 2 ** 12))
def test_thresholds_vs_exact_rationals(p, q):
    T = oracle.thresholds(p, q)
    assert T == pyoracle.thresholds(p, q)
    mn = min(Fraction(p), Fraction(1), Fraction(q))
    for c, t in zip((Fraction(p), Fraction(1), Fraction(q)), T):
        exact = Fraction(2 ** 32) * mn / c
        # one IEEE division (mn / c) then an exact scaling: within 1 of the exact floor,
        # and equal to it whenever mn / c is exactly representable
        assert abs(t - math.floor(exact)) <= 1
        assert 1 <= t <= 2 ** 32
        if (mn / c).denominator & ((mn / c).denominator - 1) == 0:
            assert t == math.floor(exact)
    assert max(T) == 2 ** 32   # the largest class always accepts


# --------------------------------------------------------------------------- prefix sums
def test_prefix_matches_numpy_cumsum_per_row():
    g = tiny_graph(5, 40, 0.2, weighted=True, max_w=1000)
    n, off, col, w = g.numpy()
    cw = oracle.prefix(n, off, w)
    for v in range(n):
        a, b = int(off[v]), int(off[v + 1])
        assert np.array_equal(cw[a:b], np.cumsum(w[a:b].astype(np.uint64)))
    cw1 = oracle.prefix(n, off, None)
    for v in range(n):
        a, b = int(off[v]), int(off[v + 1])
        assert np.array_equal(cw1[a:b], np.arange(1, b - a + 1, dtype=np.uint64))


# --------------------------------------------------------------------------- C vs Python
@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(seed=st.integers(0, 10 ** 6), n=st.integers(1, 14), dens=st.floats(0.0, 0.7),
       directed=st.booleans(), weighted=st.booleans(),
       p=st.sampled_from([0.25, 0.5, 1.0, 2.0, 4.0, 0.3]), q=st.sampled_from([0.25, 0.5, 1.0, 2.0, 4.0, 3.0]),
       L=st.sampled_from([1, 2, 3, 7, 17]), mode=st.sampled_from(["first_order", "node2vec"]),
       base=st.sampled_from([0, 5, 2 ** 32 - 3, 2 ** 40]))
def test_c_oracle_equals_python_transliteration(seed, n, dens, directed, weighted, p, q, L, mode, base):
    g = tiny_graph(seed, n, dens, directed=directed, weighted=weighted, self_loops=directed)
    nn, off, col, w = g.numpy()
    starts = np.array(list(range(n)) + [n, n + 5, 2 ** 32 - 1], dtype=np.uint32)
    out, steps = Oracle(nn, off, col, w).walks(starts, L, mode=mode, p=p, q=q, seed=seed, base=base)
    pg = pyoracle.PyGraph(nn, off, col, w)
    tot = 0
    for i, s in enumerate(starts):
        row, st_ = pg.walk(int(s), base + i, L, mode, p, q, seed)
        assert out[i].tolist() == row
        tot += st_
    assert tot == steps

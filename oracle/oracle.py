"""ctypes wrapper around ``oracle/grape_oracle.c`` — TEST INFRASTRUCTURE ONLY.

Argument marshalling only; all arithmetic is in the C file (each function
there cites the PAPER.md / SURVEY.md §8(c) passage it follows).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

PAD = 0xFFFFFFFF
_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "grape_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build_oracle(force: bool = False) -> str:
    """Compile grape_oracle.c with gcc (plain C99 + __int128, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=gnu99", "-fPIC", "-shared", "-ffp-contract=off",
            "-fno-fast-math", "-Wall", "-o", tmp, _SRC, "-lm",
        ])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_oracle())
            lib.oracle_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
            lib.oracle_philox4x32_10.restype = None
            lib.oracle_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                        ctypes.c_uint32, _u32p]
            lib.oracle_draw.restype = None
            lib.oracle_bounded.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
            lib.oracle_bounded.restype = ctypes.c_uint64
            lib.oracle_thresholds.argtypes = [ctypes.c_double, ctypes.c_double, _u64p]
            lib.oracle_thresholds.restype = ctypes.c_int
            lib.oracle_prefix.argtypes = [ctypes.c_uint32, _u64p, _u32p, _u64p]
            lib.oracle_prefix.restype = None
            lib.oracle_upper_bound.argtypes = [_u64p, ctypes.c_uint64, ctypes.c_uint64]
            lib.oracle_upper_bound.restype = ctypes.c_uint64
            lib.oracle_walks.argtypes = [
                ctypes.c_uint32, _u64p, _u32p, _u64p, _u32p, ctypes.c_uint64, ctypes.c_uint64,
                ctypes.c_uint32, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                _u32p, _u64p, _u64p]
            lib.oracle_walks.restype = ctypes.c_int
            lib.oracle_first_order_steps.argtypes = [
                _u64p, _u32p, _u64p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                ctypes.c_uint64, ctypes.c_uint64, _u32p]
            lib.oracle_first_order_steps.restype = None
            lib.oracle_node2vec_steps.argtypes = [
                _u64p, _u32p, _u64p, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                ctypes.c_uint64, _u32p, _u32p]
            lib.oracle_node2vec_steps.restype = ctypes.c_int
            lib.oracle_suss.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                        ctypes.c_uint32, _u64p]
            lib.oracle_suss.restype = None
            lib.oracle_walks_approx.argtypes = [
                ctypes.c_uint32, _u64p, _u32p, _u64p, _u32p, ctypes.c_uint64, ctypes.c_uint64,
                ctypes.c_uint32, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                ctypes.c_uint32, _u64p, _u64p, _u32p, _u64p]
            lib.oracle_walks_approx.restype = ctypes.c_int
            lib.oracle_walks_cdf.argtypes = [
                ctypes.c_uint32, _u64p, _u32p, _u64p, _u32p, ctypes.c_uint64, ctypes.c_uint64,
                ctypes.c_uint32, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, _u32p, _u64p]
            lib.oracle_walks_cdf.restype = ctypes.c_int
            lib.oracle_cdf_steps.argtypes = [
                _u64p, _u32p, _u64p, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, _u32p]
            lib.oracle_cdf_steps.restype = ctypes.c_int
            lib.oracle_walks_folded.argtypes = [
                ctypes.c_uint32, _u64p, _u32p, _u64p, _u32p, ctypes.c_uint64, ctypes.c_uint64,
                ctypes.c_uint32, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, _u32p, _u64p, _u64p]
            lib.oracle_walks_folded.restype = ctypes.c_int
            lib.oracle_folded_steps.argtypes = [
                _u64p, _u32p, _u64p, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, _u32p, _u32p]
            lib.oracle_folded_steps.restype = ctypes.c_int
            lib.oracle_rank.argtypes = [ctypes.c_uint32, _u64p, ctypes.c_uint64]
            lib.oracle_rank.restype = ctypes.c_uint32
            lib.oracle_skipgram.argtypes = [
                ctypes.c_uint32, _u64p, _u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, _u32p, _u32p, _u32p]
            lib.oracle_skipgram.restype = ctypes.c_int
            _lib = lib
    return _lib


def _p32(a):
    return None if a is None else a.ctypes.data_as(_u32p)


def _p64(a):
    return None if a is None else a.ctypes.data_as(_u64p)


def philox4x32_10(ctr, key):
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32)
    key = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _load().oracle_philox4x32_10(_p32(ctr), _p32(key), _p32(out))
    return tuple(int(v) for v in out)


def draw(seed: int, wid: int, s: int, a: int):
    out = np.zeros(4, dtype=np.uint32)
    _load().oracle_draw(seed, wid, s, a, _p32(out))
    return tuple(int(v) for v in out)


def bounded(x64: int, W: int) -> int:
    return int(_load().oracle_bounded(x64, W))


def thresholds(p: float, q: float):
    """(T_p, T_1, T_q) or None when (p, q) is rejected."""
    T = np.zeros(3, dtype=np.uint64)
    if _load().oracle_thresholds(p, q, _p64(T)) != 0:
        return None
    return tuple(int(v) for v in T)


def suss(seed: int, wid: int, s: int, n: int, k: int) -> np.ndarray:
    """The k SUSS candidate indices of step s of walk wid at a node of degree n > k."""
    idx = np.zeros(k, dtype=np.uint64)
    _load().oracle_suss(seed, wid, s, n, k, _p64(idx))
    return idx


def prefix(n: int, off: np.ndarray, w: np.ndarray | None) -> np.ndarray:
    off = np.ascontiguousarray(off, dtype=np.uint64)
    m = int(off[-1])
    cw = np.zeros(max(m, 1), dtype=np.uint64)
    if w is not None:
        w = np.ascontiguousarray(w, dtype=np.uint32)
    _load().oracle_prefix(n, _p64(off), _p32(w), _p64(cw))
    return cw[:m]


def upper_bound(row: np.ndarray, r: int) -> int:
    row = np.ascontiguousarray(row, dtype=np.uint64)
    return int(_load().oracle_upper_bound(_p64(row), len(row), r))


class Oracle:
    """A host CSR graph plus its oracle prefix sums (weights None = unweighted)."""

    def __init__(self, n: int, off: np.ndarray, col: np.ndarray, w: np.ndarray | None = None):
        self.n = int(n)
        self.off = np.ascontiguousarray(off, dtype=np.uint64)
        self.col = np.ascontiguousarray(col, dtype=np.uint32)
        if len(self.col) == 0:
            self.col = np.zeros(1, dtype=np.uint32)
        self.weighted = w is not None
        self.cw = prefix(self.n, self.off, w) if self.weighted else None
        if self.cw is not None and len(self.cw) == 0:
            self.cw = np.zeros(1, dtype=np.uint64)

    def walks(self, starts, L: int, *, mode: str = "node2vec", p: float = 1.0, q: float = 1.0,
              seed: int = 42, base: int = 0, with_attempts: bool = False):
        """Walk matrix u32[len(starts), L]; also (steps, attempts) counters."""
        starts = np.ascontiguousarray(starts, dtype=np.uint32)
        nw = len(starts)
        out = np.empty((nw, L), dtype=np.uint32)
        steps = ctypes.c_uint64(0)
        att = ctypes.c_uint64(0)
        m = 0 if mode in ("first_order", "first-order", 0) else 1
        rc = _load().oracle_walks(self.n, _p64(self.off), _p32(self.col), _p64(self.cw),
                                  _p32(starts), nw, base, L, m, float(p), float(q), seed,
                                  out.ctypes.data_as(_u32p), ctypes.byref(steps),
                                  ctypes.byref(att))
        if rc != 0:
            raise ValueError(f"oracle rejected p={p} q={q}")
        if with_attempts:
            return out, int(steps.value), int(att.value)
        return out, int(steps.value)

    def walks_approx(self, starts, L: int, k: int, *, mode: str = "node2vec", p: float = 1.0,
                     q: float = 1.0, seed: int = 42, base: int = 0):
        """Approximated walks with degree threshold k (SUSS, §8(f) f1); (matrix, steps)."""
        starts = np.ascontiguousarray(starts, dtype=np.uint32)
        nw = len(starts)
        out = np.empty((nw, L), dtype=np.uint32)
        steps = ctypes.c_uint64(0)
        cand = np.zeros(max(k, 1), dtype=np.uint64)
        ccum = np.zeros(max(k, 1), dtype=np.uint64)
        m = 0 if mode in ("first_order", "first-order", 0) else 1
        rc = _load().oracle_walks_approx(self.n, _p64(self.off), _p32(self.col), _p64(self.cw),
                                         _p32(starts), nw, base, L, m, float(p), float(q), seed, k,
                                         _p64(cand), _p64(ccum), out.ctypes.data_as(_u32p),
                                         ctypes.byref(steps))
        if rc != 0:
            raise ValueError(f"oracle rejected p={p} q={q}")
        return out, int(steps.value)

    def walks_cdf(self, starts, L: int, *, p: float = 1.0, q: float = 1.0, seed: int = 42, base: int = 0):
        """Node2vec walks with the paper's CDF sampler (§8(f) f2); (matrix, steps)."""
        starts = np.ascontiguousarray(starts, dtype=np.uint32)
        nw = len(starts)
        out = np.empty((nw, L), dtype=np.uint32)
        steps = ctypes.c_uint64(0)
        rc = _load().oracle_walks_cdf(self.n, _p64(self.off), _p32(self.col), _p64(self.cw), _p32(starts), nw,
                                      base, L, float(p), float(q), seed, out.ctypes.data_as(_u32p),
                                      ctypes.byref(steps))
        if rc != 0:
            raise ValueError(f"oracle rejected p={p} q={q}")
        return out, int(steps.value)

    def rank(self, e: int) -> int:
        """The node whose row holds arc index e (P:405's Elias-Fano rank; §8(f) f3)."""
        return int(_load().oracle_rank(self.n, _p64(self.off), int(e)))

    def skipgram(self, walks, window: int, negatives: int, *, seed: int = 42, base: int = 0):
        """SkipGram pairs and scale-free negatives of a walk matrix (§8(f) f3):
        (centers u32[S], contexts u32[S], negs u32[S, K]), S = rows * L * 2 * window."""
        walks = np.ascontiguousarray(walks, dtype=np.uint32)
        nw, L = walks.shape
        S = nw * L * 2 * window
        c = np.empty(S, dtype=np.uint32)
        x = np.empty(S, dtype=np.uint32)
        ng = np.empty((S, negatives), dtype=np.uint32)
        _load().oracle_skipgram(self.n, _p64(self.off), walks.ctypes.data_as(_u32p), nw, base, L, window,
                                negatives, seed, c.ctypes.data_as(_u32p), x.ctypes.data_as(_u32p),
                                ng.ctypes.data_as(_u32p))
        return c, x, ng

    def walks_folded(self, starts, L: int, *, p: float = 1.0, q: float = 1.0, seed: int = 42, base: int = 0,
                     with_attempts: bool = False):
        """Node2vec walks with the outlier-folded rejection rule (§8(f) f2)."""
        starts = np.ascontiguousarray(starts, dtype=np.uint32)
        nw = len(starts)
        out = np.empty((nw, L), dtype=np.uint32)
        steps = ctypes.c_uint64(0)
        att = ctypes.c_uint64(0)
        rc = _load().oracle_walks_folded(self.n, _p64(self.off), _p32(self.col), _p64(self.cw), _p32(starts), nw,
                                         base, L, float(p), float(q), seed, out.ctypes.data_as(_u32p),
                                         ctypes.byref(steps), ctypes.byref(att))
        if rc != 0:
            raise ValueError(f"oracle rejected p={p} q={q}")
        if with_attempts:
            return out, int(steps.value), int(att.value)
        return out, int(steps.value)

    def folded_steps(self, t: int, v: int, s: int, wid0: int, count: int, p: float, q: float, seed: int = 42):
        x = np.empty(count, dtype=np.uint32)
        a = np.empty(count, dtype=np.uint32)
        rc = _load().oracle_folded_steps(_p64(self.off), _p32(self.col), _p64(self.cw), float(p), float(q), seed,
                                         t, v, s, wid0, count, _p32(x), _p32(a))
        if rc != 0:
            raise ValueError(f"oracle rejected p={p} q={q}")
        return x, a

    def cdf_steps(self, t: int, v: int, s: int, wid0: int, count: int, p: float, q: float, seed: int = 42):
        x = np.empty(count, dtype=np.uint32)
        rc = _load().oracle_cdf_steps(_p64(self.off), _p32(self.col), _p64(self.cw), float(p), float(q), seed,
                                      t, v, s, wid0, count, _p32(x))
        if rc != 0:
            raise ValueError(f"oracle rejected p={p} q={q}")
        return x

    def first_order_steps(self, v: int, s: int, wid0: int, count: int, seed: int = 42):
        x = np.empty(count, dtype=np.uint32)
        _load().oracle_first_order_steps(_p64(self.off), _p32(self.col), _p64(self.cw), seed,
                                         v, s, wid0, count, _p32(x))
        return x

    def node2vec_steps(self, t: int, v: int, s: int, wid0: int, count: int, p: float, q: float,
                       seed: int = 42):
        x = np.empty(count, dtype=np.uint32)
        a = np.empty(count, dtype=np.uint32)
        rc = _load().oracle_node2vec_steps(_p64(self.off), _p32(self.col), _p64(self.cw),
                                           float(p), float(q), seed, t, v, s, wid0, count,
                                           _p32(x), _p32(a))
        if rc != 0:
            raise ValueError(f"oracle rejected p={p} q={q}")
        return x, a


def walks(n, off, col, w, starts, L, **kw):
    return Oracle(n, off, col, w).walks(starts, L, **kw)


def first_order_steps(n, off, col, w, v, s, wid0, count, seed=42):
    return Oracle(n, off, col, w).first_order_steps(v, s, wid0, count, seed)


def node2vec_steps(n, off, col, w, t, v, s, wid0, count, p, q, seed=42):
    return Oracle(n, off, col, w).node2vec_steps(t, v, s, wid0, count, p, q, seed)

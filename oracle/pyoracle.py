"""Pure-Python transliteration of ``grape_oracle.c`` — TEST INFRASTRUCTURE ONLY.

Written independently of the C file from the same rules,
with Python big integers for the 128-bit product and ``bisect`` for the
searches, for tiny graphs only.  Its purpose is to catch implementation slips
in the C oracle (overflow, word order, off-by-one) by bit-exact comparison;
the *rules themselves* are pinned by the statistical / closed-form tests.

The ``mutation`` knob builds deliberately wrong samplers for the test-power
checks (tests/test_oracle_stats.py): a statistical pin that cannot tell these
apart from the correct rule has no power.
"""
from __future__ import annotations

import bisect
from fractions import Fraction
import math

PAD = 0xFFFFFFFF
NONE = 0xFFFFFFFF
_MASK32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = (int(v) & _MASK32 for v in ctr)
    k0, k1 = (int(v) & _MASK32 for v in key)
    for rnd in range(10):
        if rnd:
            k0 = (k0 + 0x9E3779B9) & _MASK32
            k1 = (k1 + 0xBB67AE85) & _MASK32
        p0 = 0xD2511F53 * c0
        p1 = 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & _MASK32, p1 & _MASK32, \
                         ((p0 >> 32) ^ c3 ^ k1) & _MASK32, p0 & _MASK32
    return c0, c1, c2, c3


def draw(seed, wid, s, a):
    return philox4x32_10((wid & _MASK32, wid >> 32, s, a), (seed & _MASK32, seed >> 32))


def bounded(x64, W):
    return (x64 * W) >> 64


def thresholds(p, q):
    if not (p > 0 and q > 0 and math.isfinite(p) and math.isfinite(q)):
        return None
    mn, mx = min(p, 1.0, q), max(p, 1.0, q)
    if mx / mn > 2.0 ** 24:
        return None
    return tuple(int(math.floor(math.ldexp(mn / c, 32))) for c in (p, 1.0, q))


class PyGraph:
    def __init__(self, n, off, col, w=None):
        self.n = int(n)
        self.off = [int(v) for v in off]
        self.col = [int(v) for v in col]
        self.rows = [self.col[self.off[v]:self.off[v + 1]] for v in range(self.n)]
        self.cw = None
        if w is not None:
            w = [int(v) for v in w]
            self.cw = []
            for v in range(self.n):
                acc, row = 0, []
                for e in range(self.off[v], self.off[v + 1]):
                    acc += w[e]
                    row.append(acc)
                self.cw.append(row)

    def propose(self, v, x64):
        row = self.rows[v]
        if self.cw is None:
            return row[bounded(x64, len(row))]
        c = self.cw[v]
        r = bounded(x64, c[-1])
        return row[bisect.bisect_right(c, r)]

    def member(self, t, x):
        row = self.rows[t]
        i = bisect.bisect_left(row, x)
        return i < len(row) and row[i] == x

    def node2vec_step(self, T, seed, wid, s, t, v, mutation=None):
        a = 0
        while True:
            o = draw(seed, wid, s, a + (1 if mutation == "attempt+1" else 0))
            x = self.propose(v, (o[1] << 32) | o[0])
            if x == t and mutation != "drop-return":
                thr = T[0]
            elif self.member(t, x):
                thr = T[2] if mutation == "swap-1-q" else T[1]
            else:
                thr = T[1] if mutation == "swap-1-q" else T[2]
            a += 1
            if o[2] < thr:
                return x, a

    # ---- approximated walks (SUSS, §8(f) f1) ----
    def suss(self, seed, wid, s, n, k):
        """k sorted unique candidate positions, one uniform draw per bucket
        [floor(b n / k), floor((b+1) n / k)); bucket b's 64-bit draw is half of the
        Philox block with counter (wid, s, 2^31 + b // 2)."""
        out = []
        for b in range(k):
            lo, hi = b * n // k, (b + 1) * n // k
            o = draw(seed, wid, s, 0x80000000 | (b // 2))
            h = (o[1] << 32 | o[0]) if b % 2 == 0 else (o[3] << 32 | o[2])
            out.append(lo + bounded(h, hi - lo))
        return out

    def propose_among(self, v, cand, x64):
        row = self.rows[v]
        if self.cw is None:
            ws = [1] * len(cand)
        else:
            c = self.cw[v]
            ws = [c[j] - (c[j - 1] if j else 0) for j in cand]
        cum, acc = [], 0
        for wj in ws:
            acc += wj
            cum.append(acc)
        r = bounded(x64, acc)
        return row[cand[bisect.bisect_right(cum, r)]]

    def walk_approx(self, start, wid, L, k, mode="node2vec", p=1.0, q=1.0, seed=42):
        row = [PAD] * L
        if start >= self.n or L == 0:
            return row, 0
        T = thresholds(p, q) if mode == "node2vec" else None
        row[0] = start
        t, v, steps = NONE, start, 0
        for s in range(1, L):
            n = len(self.rows[v])
            if n == 0:
                break
            cand = self.suss(seed, wid, s, n, k) if 0 < k < n else None

            def prop(x64):
                return self.propose(v, x64) if cand is None else self.propose_among(v, cand, x64)
            if mode == "first_order" or t == NONE:
                o = draw(seed, wid, s, 0)
                x = prop((o[1] << 32) | o[0])
            else:
                a = 0
                while True:
                    o = draw(seed, wid, s, a)
                    x = prop((o[1] << 32) | o[0])
                    thr = T[0] if x == t else (T[1] if self.member(t, x) else T[2])
                    a += 1
                    if o[2] < thr:
                        break
            row[s] = x
            steps += 1
            t, v = v, x
        return row, steps

    # ---- outlier-folded rejection (§8(f) f2) ----
    def folded_step(self, T, seed, wid, s, t, v):
        E = max(T[1], T[2])
        X = T[0] - E if T[0] > E else 0
        A = [-(-(min(tc, E) << 32) // E) for tc in T]          # ceil(min(T_c, E) 2^32 / E)
        row = self.rows[v]
        if self.cw is None:
            W, wt = len(row), (1 if t in row else 0)
        else:
            c = self.cw[v]
            W = c[-1]
            wt = 0
            for i, x in enumerate(row):
                if x == t:
                    wt = c[i] - (c[i - 1] if i else 0)
        N = wt * X
        M = W * E + N
        a = 0
        while True:
            o = draw(seed, wid, s, a)
            a += 1
            if N > 0 and o[3] * M < (N << 32):
                return t, a
            x = self.propose(v, (o[1] << 32) | o[0])
            thr = A[0] if x == t else (A[1] if self.member(t, x) else A[2])
            if o[2] < thr:
                return x, a

    def walk_folded(self, start, wid, L, p=1.0, q=1.0, seed=42):
        row = [PAD] * L
        if start >= self.n or L == 0:
            return row, 0
        T = thresholds(p, q)
        row[0] = start
        t, v, steps = NONE, start, 0
        for s in range(1, L):
            if not self.rows[v]:
                break
            if t == NONE:
                o = draw(seed, wid, s, 0)
                x = self.propose(v, (o[1] << 32) | o[0])
            else:
                x, _ = self.folded_step(T, seed, wid, s, t, v)
            row[s] = x
            steps += 1
            t, v = v, x
        return row, steps

    # ---- the paper's CDF sampler (§8(f) f2; P:507-511 steps 1-4) ----
    def cdf_step(self, T, seed, wid, s, t, v):
        row = self.rows[v]
        if self.cw is None:
            ws = [1] * len(row)
        else:
            c = self.cw[v]
            ws = [c[i] - (c[i - 1] if i else 0) for i in range(len(c))]
        pis = [wx * (T[0] if x == t else (T[1] if self.member(t, x) else T[2])) for x, wx in zip(row, ws)]
        o = draw(seed, wid, s, 0)
        r = ((o[1] << 32 | o[0]) * sum(pis)) >> 64       # exact big-integer product
        acc = 0
        for x, pi in zip(row, pis):
            acc += pi
            if acc > r:
                return x
        raise AssertionError("unreachable")

    def walk_cdf(self, start, wid, L, p=1.0, q=1.0, seed=42):
        row = [PAD] * L
        if start >= self.n or L == 0:
            return row, 0
        T = thresholds(p, q)
        row[0] = start
        t, v, steps = NONE, start, 0
        for s in range(1, L):
            if not self.rows[v]:
                break
            if t == NONE:
                o = draw(seed, wid, s, 0)
                x = self.propose(v, (o[1] << 32) | o[0])
            else:
                x = self.cdf_step(T, seed, wid, s, t, v)
            row[s] = x
            steps += 1
            t, v = v, x
        return row, steps

    def walk(self, start, wid, L, mode="node2vec", p=1.0, q=1.0, seed=42, mutation=None):
        row = [PAD] * L
        if start >= self.n or L == 0:
            return row, 0
        T = thresholds(p, q) if mode == "node2vec" else None
        if mode == "node2vec" and T is None:
            raise ValueError("bad p/q")
        row[0] = start
        t, v, steps = NONE, start, 0
        for s in range(1, L):
            if not self.rows[v]:
                break
            if mode == "first_order" or t == NONE:
                o = draw(seed, wid, s, 0)
                x = self.propose(v, (o[1] << 32) | o[0])
            else:
                x, _ = self.node2vec_step(T, seed, wid, s, t, v, mutation)
            row[s] = x
            steps += 1
            t, v = v, x
        return row, steps


def skipgram(g: PyGraph, walks, window, K, seed=42, base=0):
    """SkipGram pairs + scale-free negatives (§8(f) f3): lists (centers, contexts,
    negatives-per-slot), slot order (row, i, j = -w..-1, 1..w)."""
    m = g.off[-1] if g.n else 0
    centers, contexts, negs = [], [], []
    for r, row in enumerate(walks):
        L = len(row)
        for i in range(L):
            for j in list(range(-window, 0)) + list(range(1, window + 1)):
                o = j + window if j < 0 else j + window - 1
                c = i + j
                ok = 0 <= c < L and row[i] != PAD and row[c] != PAD
                centers.append(row[i] if ok else PAD)
                contexts.append(row[c] if ok else PAD)
                slot = ((base + r) * L + i) * 2 * window + o
                ks = []
                for k in range(K):
                    if not ok or m == 0:
                        ks.append(PAD)
                        continue
                    d = draw(seed, slot, 0xFFFFFFFF, k // 2)      # two negatives per block
                    e = bounded((d[3] << 32 | d[2]) if k % 2 else (d[1] << 32 | d[0]), m)
                    ks.append(bisect.bisect_right(g.off, e) - 1)   # the row holding arc e
                negs.append(ks)
    return centers, contexts, negs


def eq1_law(g: PyGraph, t, v, p, q, weights_of=None):
    """Exact node2vec step law from Eq.1 as Fractions:
    pi_vx = alpha_pq(t,x) w_vx, alpha = 1/p (x == t), 1 (x in N(t)), 1/q (else)."""
    p, q = Fraction(p), Fraction(q)
    row = g.rows[v]
    if g.cw is None:
        w = [1] * len(row)
    else:
        c = g.cw[v]
        w = [c[0]] + [c[i] - c[i - 1] for i in range(1, len(c))]
    pis = []
    for x, wx in zip(row, w):
        if x == t:
            alpha = 1 / p
        elif g.member(t, x):
            alpha = Fraction(1)
        else:
            alpha = 1 / q
        pis.append(alpha * wx)
    tot = sum(pis)
    return {x: pi / tot for x, pi in zip(row, pis)}

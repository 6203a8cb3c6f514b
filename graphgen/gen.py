"""Counter-based graph generators (torch ops; identical results on CPU and CUDA)."""
from __future__ import annotations

from dataclasses import dataclass
import math

import numpy as np
import torch

_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def _s64(v: int) -> int:
    """Python int -> the int64 with the same 64 bits."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 bit patterns (wrapping arithmetic)."""
    x = x + _s64(_GOLDEN)
    x = (x ^ _srl(x, 30)) * _s64(_M1)
    x = (x ^ _srl(x, 27)) * _s64(_M2)
    return x ^ _srl(x, 31)


def hash3(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """64 random bits for (seed, stream, idx) — keyed by all three."""
    k = splitmix64(torch.tensor([_s64(seed * 0x100000001B3 + stream)], dtype=torch.int64,
                                device=idx.device))
    return splitmix64(idx.to(torch.int64) ^ k)


def _hi32(h: torch.Tensor) -> torch.Tensor:
    return _srl(h, 32)


def _unit53(h: torch.Tensor) -> torch.Tensor:
    """Exact double in [0, 1) from the top 53 bits."""
    return _srl(h, 11).to(torch.float64) * (2.0 ** -53)


@dataclass
class CSR:
    """Host or device CSR: off int64[n+1], col int32 view of u32[m], w int32 view of u32[m] or None.

    torch has no arithmetic on uint32 / uint64, so the arrays are stored as
    int64 / int32 with the same bit patterns as the C-ABI's u64 / u32 arrays.
    """
    n: int
    off: torch.Tensor
    col: torch.Tensor
    w: torch.Tensor | None
    symmetric: bool
    name: str = ""

    @property
    def m(self) -> int:
        return int(self.col.numel())

    def to(self, device) -> "CSR":
        return CSR(self.n, self.off.to(device), self.col.to(device),
                   None if self.w is None else self.w.to(device), self.symmetric, self.name)

    def numpy(self):
        """(n, off u64, col u32, w u32|None) numpy views for the oracle."""
        off = self.off.cpu().numpy().astype(np.uint64)
        col = self.col.cpu().numpy().view(np.uint32)
        w = None if self.w is None else self.w.cpu().numpy().view(np.uint32)
        return self.n, off, col, w

    def nbytes(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in (self.off, self.col, self.w)
                   if t is not None)


def csr_from_arcs(n: int, src: torch.Tensor, dst: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Sort arcs by (src, dst), drop duplicates; return (off int64[n+1], col int32[m])."""
    key = src.to(torch.int64) * n + dst.to(torch.int64)
    key = torch.unique(key, sorted=True)
    s = torch.div(key, n, rounding_mode="floor")
    col = (key - s * n).to(torch.int32)
    cnt = torch.bincount(s, minlength=n)
    off = torch.zeros(n + 1, dtype=torch.int64, device=key.device)
    off[1:] = torch.cumsum(cnt, 0)
    return off, col


def _csr_from_sorted_keys(n: int, key: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """CSR of sorted unique arc keys src * n + dst."""
    src = torch.div(key, n, rounding_mode="floor")
    col = (key - src * n).to(torch.int32)
    off = torch.zeros(n + 1, dtype=torch.int64, device=key.device)
    off[1:] = torch.cumsum(torch.bincount(src, minlength=n), 0)
    return off, col


# torch's CUB-backed sort / unique refuse more than 2^31 - 1 elements: above this,
# work by key-value ranges (bucket b holds the keys in [b K / B, (b+1) K / B)), each
# bucket sorted on its own; the concatenation is the same sorted array.
_BIG = (1 << 31) - (1 << 20)


def _by_ranges(x: torch.Tensor, kmax: int, fn, buckets: int = 32) -> torch.Tensor:
    out = []
    for j in range(buckets):
        lo, hi = kmax * j // buckets, kmax * (j + 1) // buckets
        sel = x[(x >= lo) & (x < hi)]
        if sel.numel():
            out.append(fn(sel))
        del sel
    return torch.cat(out) if out else x[:0]


def _sorted_unique(key: torch.Tensor, kmax: int) -> torch.Tensor:
    if key.numel() <= _BIG:
        return torch.unique(key, sorted=True)
    return _by_ranges(key, kmax, lambda s: torch.unique(s, sorted=True))


def _sorted(key: torch.Tensor, kmax: int) -> torch.Tensor:
    if key.numel() <= _BIG:
        return torch.sort(key).values
    return _by_ranges(key, kmax, lambda s: torch.sort(s).values)


def _bincount_rows(key: torch.Tensor, n: int, chunk: int = 1 << 28) -> torch.Tensor:
    cnt = torch.zeros(n, dtype=torch.int64, device=key.device)
    for lo in range(0, key.numel(), chunk):
        cnt += torch.bincount(torch.div(key[lo:lo + chunk], n, rounding_mode="floor"), minlength=n)
    return cnt


def _csr_symmetric(n: int, ckey: torch.Tensor, chunk: int = 1 << 28) -> tuple[torch.Tensor, torch.Tensor]:
    """Symmetric CSR from sorted unique canonical keys a * n + b (a < b): every edge
    gives arcs a->b and b->a.  The reversed keys are sorted once and merged by rank
    (searchsorted), so no sort ever holds all 2m arcs (and the merge runs in chunks)."""
    m1 = ckey.numel()
    rkey = torch.empty_like(ckey)
    for lo in range(0, m1, chunk):
        ck = ckey[lo:lo + chunk]
        a = torch.div(ck, n, rounding_mode="floor")
        rkey[lo:lo + chunk] = (ck - a * n) * n + a
        del a
    rkey = _sorted(rkey, n * n)
    col = torch.empty(2 * m1, dtype=torch.int32, device=ckey.device)
    for src, other in ((ckey, rkey), (rkey, ckey)):
        for lo in range(0, m1, chunk):
            s = src[lo:lo + chunk]
            pos = torch.arange(lo, lo + s.numel(), device=ckey.device) + torch.searchsorted(other, s)
            col[pos] = (s % n).to(torch.int32)
            del pos
    cnt = _bincount_rows(ckey, n, chunk) + _bincount_rows(rkey, n, chunk)
    off = torch.zeros(n + 1, dtype=torch.int64, device=ckey.device)
    off[1:] = torch.cumsum(cnt, 0)
    return off, col


def _arc_rows(off: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """Source node of arcs [lo, hi)."""
    e = torch.arange(lo, hi, device=off.device, dtype=torch.int64)
    return torch.searchsorted(off, e, right=True) - 1


def _permutation(n: int, seed: int, device) -> torch.Tensor:
    """Seeded random permutation of [0, n): stable argsort of per-label hashes."""
    h = hash3(seed, 0x5045524D, torch.arange(n, device=device, dtype=torch.int64))
    return torch.argsort(h, stable=True)


def _sym_weights(n: int, a: torch.Tensor, b: torch.Tensor, seed: int, kind: str, K: int) -> torch.Tensor:
    """Per-undirected-edge weight, keyed by the canonical (min, max) pair so both
    arcs of an edge get the same value.  kind 'uniform': U{1..K}."""
    lo, hi = torch.minimum(a, b).to(torch.int64), torch.maximum(a, b).to(torch.int64)
    h = hash3(seed, 0x57454947, lo * n + hi)
    if kind == "uniform":
        return (1 + ((_hi32(h) * K) >> 32)).to(torch.int32)
    raise ValueError(kind)


def _geometric_weights(key: torch.Tensor, seed: int, mean: float) -> torch.Tensor:
    """Geometric weights on {1, 2, ...} with P(w = k) = (1-r)^(k-1) r, r = 1/mean,
    drawn by inverse CDF against a table of survival thresholds
    S_k = floor(2^53 (1-r)^k) computed here once in Python doubles (host-only
    constants), so CPU and CUDA compare the same integers."""
    r = 1.0 / mean
    kmax = 1 + int(math.ceil(math.log(2.0 ** -53) / math.log(1.0 - r)))
    surv = [int(math.floor((1.0 - r) ** k * 2.0 ** 53)) for k in range(1, kmax + 1)]
    # w = 1 + #{k >= 1 : U53 < S_k}   (U53 uniform on [0, 2^53)); S_k decreasing.
    table = torch.tensor(surv[::-1], dtype=torch.int64, device=key.device)  # increasing
    u = _srl(hash3(seed, 0x47454F4D, key), 11)
    cnt_ge = torch.searchsorted(table, u, right=True)  # #{S_k <= u}
    return (1 + (len(surv) - cnt_ge)).to(torch.int32)


def chung_lu(n: int, m_target: int, *, seed: int, weights: int | None = None,
             device="cpu", chunk: int = 1 << 26, name: str = "") -> CSR:
    """Undirected Chung-Lu power-law graph, exponent gamma = 2.5.

    Expected-degree weights omega_i ∝ (i+1)^(-1/(gamma-1)) = (i+1)^(-2/3).
    Each of m_target pairs draws both endpoints i.i.d. ∝ omega through the
    inverse CDF of the continuous density x^(-2/3) on [1, n+1):
        x = (1 + U c)^3,  c = (n+1)^(1/3) - 1,  i = floor(x) - 1.
    Labels are then permuted (hubs scattered), self-loops dropped, pairs
    canonicalised and deduplicated, mirrored, and rows sorted.
    weights=K gives U{1..K} per undirected edge, mirrored."""
    c = (n + 1.0) ** (1.0 / 3.0) - 1.0
    perm = _permutation(n, seed, device)
    keys = []
    for lo in range(0, m_target, chunk):
        k = torch.arange(lo, min(m_target, lo + chunk), device=device, dtype=torch.int64)
        ends = []
        for stream in (1, 2):
            u = _unit53(hash3(seed, stream, k))
            y = u * c
            y = y + 1.0
            x = (y * y) * y
            i = x.floor().to(torch.int64) - 1
            i = i.clamp_(0, n - 1)
            ends.append(perm[i])
        a, b = ends
        keep = a != b
        a, b = a[keep], b[keep]
        keys.append(torch.minimum(a, b) * n + torch.maximum(a, b))
    key = torch.cat(keys)
    del keys
    key = _sorted_unique(key, n * n)
    off, col = _csr_symmetric(n, key)
    del key
    w = None
    if weights is not None:
        w = torch.empty_like(col)
        m = col.numel()
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            w[lo:hi] = _sym_weights(n, _arc_rows(off, lo, hi), col[lo:hi].to(torch.int64), seed, "uniform",
                                    weights)
    return CSR(n, off, col, w, True, name or f"chung_lu(n={n},m={m_target})")


def rmat(scale: int, edge_factor: int, *, seed: int, a=0.57, b=0.19, c=0.19,
         symmetric: bool = True, weights=None, device="cpu", chunk: int = 1 << 25,
         sink_fraction: float | None = None, name: str = "") -> CSR:
    """R-MAT (Graph500-style quadrant recursion, no noise).

    ef * 2^scale samples; at each of `scale` levels one 32-bit draw u picks the
    quadrant: u < A -> (0,0), < A+B -> (0,1), < A+B+C -> (1,0), else (1,1),
    with A = floor(a 2^32) etc.  Labels permuted, self-loops dropped, deduped;
    symmetric=True mirrors every edge.  weights=('geometric', mean) draws a
    geometric weight per arc (directed) / per edge (symmetric)."""
    n = 1 << scale
    A = int(a * 2 ** 32)
    AB = int((a + b) * 2 ** 32)
    ABC = int((a + b + c) * 2 ** 32)
    perm = _permutation(n, seed, device)
    total = edge_factor * n
    keys = []
    for lo in range(0, total, chunk):
        k = torch.arange(lo, min(total, lo + chunk), device=device, dtype=torch.int64)
        s = torch.zeros_like(k)
        d = torch.zeros_like(k)
        for lev in range(scale):
            u = _hi32(hash3(seed, 0x100 + lev, k))
            row_bit = (u >= AB).to(torch.int64)
            col_bit = (((u >= A) & (u < AB)) | (u >= ABC)).to(torch.int64)
            s = (s << 1) | row_bit
            d = (d << 1) | col_bit
        s, d = perm[s], perm[d]
        keep = s != d
        s, d = s[keep], d[keep]
        if symmetric:
            keys.append(torch.minimum(s, d) * n + torch.maximum(s, d))
        else:
            keys.append(s * n + d)
    key = torch.unique(torch.cat(keys), sorted=True)
    del keys
    if symmetric:
        off, col = _csr_symmetric(n, key)
    else:
        if sink_fraction is not None:
            key = _fix_sinks(n, key, seed, sink_fraction)
        off, col = _csr_from_sorted_keys(n, key)
    del key
    w = None
    if weights is not None:
        kind, mean = weights
        assert kind == "geometric"
        w = torch.empty_like(col)
        m = col.numel()
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            rows = _arc_rows(off, lo, hi)
            cc = col[lo:hi].to(torch.int64)
            ekey = (torch.minimum(rows, cc) * n + torch.maximum(rows, cc)) if symmetric else rows * n + cc
            w[lo:hi] = _geometric_weights(ekey, seed, mean)
    return CSR(n, off, col, w, symmetric, name or f"rmat(scale={scale},ef={edge_factor})")


def _fix_sinks(n: int, key: torch.Tensor, seed: int, fraction: float) -> torch.Tensor:
    """Directed R-MAT leaves far more out-degree-0 nodes than BASELINE configs[4]'s
    "~5% dead-end nodes".  Keep a seeded random subset of
    round(fraction * n) of the natural sinks as sinks; give every other sink one
    out-arc to col[j] for a uniformly drawn arc j (targets ∝ in-degree), redrawing
    on a self-loop.  Returns the sorted keys with the new arcs merged in."""
    device = key.device
    src = torch.div(key, n, rounding_mode="floor")
    deg = torch.bincount(src, minlength=n)
    del src
    sinks = torch.nonzero(deg == 0).flatten()
    keep = int(round(fraction * n))
    if sinks.numel() <= keep:
        return key
    order = torch.argsort(hash3(seed, 0x53494E4B, sinks), stable=True)
    fix = torch.sort(sinks[order[keep:]]).values
    m = key.numel()
    tgt = torch.full_like(fix, -1)
    for attempt in range(64):
        todo = tgt < 0
        if not bool(todo.any()):
            break
        h = hash3(seed, 0x54475400 + attempt, fix[todo])
        j = (_hi32(h) * m) >> 32
        t = key[j] % n
        t = torch.where(t == fix[todo], torch.full_like(t, -1), t)
        tgt[todo] = t
    ok = tgt >= 0
    new = torch.sort(fix[ok] * n + tgt[ok]).values
    out = torch.empty(m + new.numel(), dtype=key.dtype, device=device)
    idx = torch.arange(m, device=device)
    out[idx + torch.searchsorted(new, key)] = key
    idx = torch.arange(new.numel(), device=device)
    out[idx + torch.searchsorted(key, new)] = new
    return out


def tiny_graph(seed: int, n: int, density: float, *, directed: bool = False,
               weighted: bool = False, max_w: int = 9, self_loops: bool = False) -> CSR:
    """Small random graph for fuzz / parity tests (numpy RNG, host only)."""
    rng = np.random.default_rng(seed)
    adj = rng.random((n, n)) < density
    if not self_loops:
        np.fill_diagonal(adj, False)
    if not directed:
        adj = np.triu(adj, 1)
        adj = adj | adj.T
    wmat = rng.integers(1, max_w + 1, size=(n, n))
    if not directed:
        wmat = np.triu(wmat, 1)
        wmat = wmat + wmat.T
    src, dst = np.nonzero(adj)
    off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off)
    w = torch.from_numpy(wmat[src, dst].astype(np.int32)) if weighted else None
    return CSR(n, torch.from_numpy(off), torch.from_numpy(dst.astype(np.int32)), w,
               not directed, f"tiny(seed={seed},n={n})")


def starts_per_node(n: int, walks_per_node: int, device="cpu") -> torch.Tensor:
    """Iteration-major start list: wid = it * n + node."""
    return torch.arange(n, dtype=torch.int64, device=device).repeat(walks_per_node).to(torch.int32)

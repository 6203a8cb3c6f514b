"""paper_2110_06196_b200 — B200-native bulk random walks (GRAPE, arxiv 2110.06196).

Thin Python binding over the C-ABI in ``include/grape_walk.h`` (argument
marshalling only; every step of the walk runs in the CUDA kernels of
``libgrape_walk.so``).  PyTorch supplies device memory and streams.

    g = graph_from_csr(off, col, weights=None, device=0, symmetric=True)
    out = walks_node2vec(g, starts, L=80, p=0.5, q=2.0, seed=42)   # int32 [W, L]; PAD = -1
    out = walks_first_order(g, starts, L=32, seed=42)

``starts`` on a CUDA device -> asynchronous on the current stream, result on
the device.  ``starts`` on the CPU -> the library stages host buffers itself
(H2D / kernel / D2H pipelined in chunks) and returns a (pinned) CPU tensor.
Walk matrices are int32 tensors holding the u32 bit patterns: GRAPE_PAD
(0xFFFFFFFF) reads as -1.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _capi
from ._capi import (GRAPE_PAD, GRAPE_SYMMETRIC, GRAPE_SKIP_VALIDATION, GRAPE_NO_TABLES, GrapeError,  # noqa: F401
                    GRAPE_OK, GRAPE_EINVAL, GRAPE_ENOMEM, GRAPE_ECUDA)

_lib = _capi.load()
PAD_I32 = -1


def version() -> str:
    return _lib.grape_version().decode()


def _as_tensor(a, dtype) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype == torch.uint32:
        t = t.view(torch.int32)
    if t.dtype == torch.uint64:
        t = t.view(torch.int64)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def _check_out(out: torch.Tensor, shape, device_kind: str, what: str) -> None:
    """A caller-supplied output buffer must be exactly what the kernel writes: the library
    writes prod(shape) u32 words through its data pointer (device path) or copies them into
    it (host path), so a wrong size, dtype, layout or memory kind would corrupt memory."""
    if not torch.is_tensor(out):
        raise ValueError(f"{what} must be a torch.Tensor")
    if out.dtype not in (torch.int32, torch.uint32):
        raise ValueError(f"{what} must be int32 (u32 bit patterns), got {out.dtype}")
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"{what} must have shape {tuple(shape)}, got {tuple(out.shape)}")
    if not out.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    if device_kind == "cpu" and out.is_cuda:
        raise ValueError(f"{what} must be a host tensor (the starts are on the host)")
    if device_kind != "cpu" and (not out.is_cuda or out.device.index != int(device_kind)):
        raise ValueError(f"{what} must be on cuda:{device_kind}")


def _check_steps(steps: torch.Tensor, on_device: bool, device: int) -> None:
    """steps: a 1-element int64 counter the library adds realised transitions to (a 64-bit
    atomicAdd on the device path)."""
    if not torch.is_tensor(steps) or steps.dtype not in (torch.int64, torch.uint64) or steps.numel() != 1:
        raise ValueError("steps must be a 1-element int64 tensor")
    if not steps.is_contiguous():
        raise ValueError("steps must be contiguous")
    if on_device and (not steps.is_cuda or steps.device.index != device):
        raise ValueError(f"steps must be on cuda:{device} (the starts are device memory)")


def _stream_handle(stream, device: int, keep=()):
    """The raw cudaStream_t to launch on.  When the caller names a stream other than the
    current one, the tensors in `keep` (temporaries and outputs allocated on the current
    stream) are recorded on it, so the caching allocator cannot hand their memory to
    other work while the kernel is still queued there."""
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        if stream != torch.cuda.current_stream(device):
            for t in keep:
                if torch.is_tensor(t) and t.is_cuda:
                    t.record_stream(stream)
        return stream.cuda_stream
    return int(stream)


class Graph:
    """Owning handle of a device CSR (grape_graph*)."""

    def __init__(self, handle: int, device: int):
        self._h = ctypes.c_void_p(handle)
        self.device = device
        info = _capi.GraphInfo()
        _capi.check(_lib, _lib.grape_graph_get_info(self._h, ctypes.byref(info)), "grape_graph_get_info")
        self.info = {f: getattr(info, f) for f, _ in _capi.GraphInfo._fields_}

    @property
    def handle(self):
        return self._h

    @property
    def num_nodes(self) -> int:
        return self.info["num_nodes"]

    @property
    def num_arcs(self) -> int:
        return self.info["num_arcs"]

    def partition(self, devices) -> "Graph":
        """grape_graph_partition: split the sampling tables into len(devices) power-of-two
        parts, part j on devices[j] (the §8(f) f4 layout; default walk rules only)."""
        arr = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        _capi.check(_lib, _lib.grape_graph_partition(self._h, len(devices), arr), "grape_graph_partition")
        info = _capi.GraphInfo()
        _capi.check(_lib, _lib.grape_graph_get_info(self._h, ctypes.byref(info)), "grape_graph_get_info")
        self.info = {f: getattr(info, f) for f, _ in _capi.GraphInfo._fields_}
        return self

    def free(self) -> None:
        """grape_graph_free.  A distributed graph (graph_from_csr_dist) waits for every rank
        first: the peers read this rank's table parts until they are done walking."""
        if self._h is not None and self._h.value:
            grp = getattr(self, "_group", False)
            if grp is not False:
                import torch.distributed as dist
                if dist.is_initialized():
                    torch.cuda.synchronize(self.device)
                    dist.barrier(group=grp)
            _capi.check(_lib, _lib.grape_graph_free(self._h), "grape_graph_free")
        self._h = None

    def __del__(self):
        if getattr(self, "_group", False) is not False:
            return   # distributed: free() waits for the peers; never from a finaliser
        try:
            self.free()
        except Exception:
            pass

    def __repr__(self):
        return f"Graph({self.info})"


def graph_from_csr(row_offsets, col_indices, weights=None, *, device: int = 0,
                   symmetric: bool = False, validate: bool = True, tables: bool = True,
                   layout: dict | None = None) -> Graph:
    """grape_graph_from_csr: row_offsets u64/int64 [n+1], col_indices u32/int32 [m],
    weights u32/int32 [m] >= 1 or None.  Host or device tensors / numpy arrays.
    tables=False passes GRAPE_NO_TABLES (v3 walker, less memory, same walks);
    layout: grape_table_options fields (table_budget_bytes, record_bytes, guide_bytes,
    guide_factor, hash_h) to force parts of the table layout (grape_graph_from_csr_opts)."""
    off = _as_tensor(row_offsets, torch.int64)
    col = _as_tensor(col_indices, torch.int32)
    w = None if weights is None else _as_tensor(weights, torch.int32)
    n = off.numel() - 1
    m = col.numel()
    flags = ((GRAPE_SYMMETRIC if symmetric else 0) | (0 if validate else GRAPE_SKIP_VALIDATION)
             | (0 if tables else GRAPE_NO_TABLES))
    h = ctypes.c_void_p()
    opts = None
    if layout:
        opts = _capi.TableOptions(**layout)
    st = _lib.grape_graph_from_csr_opts(n, m, off.data_ptr(), col.data_ptr() if m else None,
                                        None if w is None else w.data_ptr(), device, flags,
                                        None if opts is None else ctypes.byref(opts), ctypes.byref(h))
    _capi.check(_lib, st, "grape_graph_from_csr")
    return Graph(h.value, device)


def graph_from_csr_dist(row_offsets, col_indices, weights=None, *, device: int, symmetric: bool = False,
                        validate: bool = True, layout: dict | None = None, table_budget_bytes: int | None = None,
                        group=None) -> Graph:
    """Distributed table build (grape_graph_dist_*; §8(f) f4): every rank of
    the torch.distributed group calls this with the same CSR; rank r owns part r of the
    sampling tables, and the returned graph walks over all parts (the peers' over
    NVLink / CUDA IPC), bit-identical to graph_from_csr's.  table_budget_bytes: table
    bytes per rank (default: the smallest free device memory over the ranks, less 10%
    of the device); the layout is chosen for world x that.  This function supplies the
    handle exchange (all_gather_object) and the barriers the C-ABI asks for; it runs
    no collective on the walk path.  Free with Graph.free() on every rank (a barrier
    first: peers read this rank's parts)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    off = _as_tensor(row_offsets, torch.int64)
    col = _as_tensor(col_indices, torch.int32)
    w = None if weights is None else _as_tensor(weights, torch.int32)
    n, m = off.numel() - 1, col.numel()
    if table_budget_bytes is None:
        with torch.cuda.device(device):
            free, total = torch.cuda.mem_get_info(device)
        mine = [int(free - 0.1 * total)]
        allv = [None] * world
        dist.all_gather_object(allv, mine[0], group=group)
        table_budget_bytes = max(1, min(allv))
    opts = _capi.TableOptions(**(layout or {}))
    opts.table_budget_bytes = int(table_budget_bytes)
    flags = (GRAPE_SYMMETRIC if symmetric else 0) | (0 if validate else GRAPE_SKIP_VALIDATION)
    h = ctypes.c_void_p()
    st = _lib.grape_graph_dist_create(n, m, off.data_ptr(), col.data_ptr() if m else None,
                                      None if w is None else w.data_ptr(), device, flags, ctypes.byref(opts),
                                      rank, world, ctypes.byref(h))
    ok = [st == GRAPE_OK]
    oks = [None] * world
    dist.all_gather_object(oks, ok[0], group=group)
    if not all(oks):   # every rank stops together (no rank left waiting in a collective)
        if st == GRAPE_OK:
            _lib.grape_graph_free(h)
            raise GrapeError(GRAPE_EINVAL, "grape_graph_dist_create failed on another rank")
        _capi.check(_lib, st, "grape_graph_dist_create")
    g = Graph.__new__(Graph)
    g._h = h
    g.device = device
    g._group = group

    def agreed(status: int, payload, what: str):
        """All-gather (status, payload) — the stage barrier — and raise on every rank if any
        rank failed, so no rank is left waiting in a collective the others never reach."""
        got = [None] * world
        dist.all_gather_object(got, (int(status), payload), group=group)
        if any(s != GRAPE_OK for s, _ in got):
            bad = next(r for r, (s, _) in enumerate(got) if s != GRAPE_OK)
            detail = _lib.grape_last_error().decode(errors="replace") if status != GRAPE_OK else ""
            _lib.grape_graph_free(h)
            g._h = None
            raise GrapeError(got[bad][0], f"{what} failed on rank {bad}" + (f": {detail}" if detail else ""))
        return [p for _, p in got]

    ex = _capi.PartExport()
    st = _lib.grape_graph_dist_export(h, ctypes.byref(ex))
    allx = agreed(st, bytes(ex), "grape_graph_dist_export")
    arr = (_capi.PartExport * world)()
    for x in allx:
        e = _capi.PartExport.from_buffer_copy(x)
        arr[e.part] = e
    agreed(_lib.grape_graph_dist_import(h, arr), None, "grape_graph_dist_import")   # every rank opened every part
    fl = ctypes.c_uint32(0)
    flags_all = 0
    for stage in range(4):
        st = _lib.grape_graph_dist_build(h, stage, ctypes.byref(fl))
        for v in agreed(st, int(fl.value), f"grape_graph_dist_build stage {stage}"):
            flags_all |= v
    st = _lib.grape_graph_dist_finish(h, flags_all)
    agreed(st, None, "grape_graph_dist_finish")
    info = _capi.GraphInfo()
    _capi.check(_lib, _lib.grape_graph_get_info(h, ctypes.byref(info)), "grape_graph_get_info")
    g.info = {f: getattr(info, f) for f, _ in _capi.GraphInfo._fields_}
    g.info["dist_part"] = rank
    return g


def _walks(fn_name, g: Graph, starts, L, args, seed, walk_id_base, out, steps, stream):
    st = _as_tensor(starts, torch.int32)
    W = st.numel()
    fn = getattr(_lib, fn_name)
    if st.is_cuda:
        if st.device.index != g.device:
            raise ValueError(f"starts on cuda:{st.device.index}, graph on cuda:{g.device}")
        with torch.cuda.device(g.device):
            if out is None:
                out = torch.empty((W, L), dtype=torch.int32, device=st.device)
            else:
                _check_out(out, (W, L), str(g.device), "out")
            if steps is not None:
                _check_steps(steps, True, g.device)
            stream = _stream_handle(stream, g.device, (st, out))
            sp = None if steps is None else steps.data_ptr()
            rc = fn(g.handle, st.data_ptr(), W, walk_id_base, L, *args, seed, out.data_ptr(), sp,
                    ctypes.c_void_p(stream))
        _capi.check(_lib, rc, fn_name)
        return out
    # host buffers: the library stages through the device itself
    if out is None:
        out = torch.empty((W, L), dtype=torch.int32, pin_memory=True)
    else:
        _check_out(out, (W, L), "cpu", "out")
    if steps is not None:
        _check_steps(steps, False, g.device)
    hs = ctypes.c_uint64(0)
    with torch.cuda.device(g.device):
        stream = _stream_handle(stream, g.device)   # host path: synchronous, nothing to record
        rc = fn(g.handle, st.data_ptr(), W, walk_id_base, L, *args, seed, out.data_ptr(),
                ctypes.byref(hs), ctypes.c_void_p(stream))
    _capi.check(_lib, rc, fn_name)
    if steps is not None:
        steps += int(hs.value)
    return out


def walks_first_order(g: Graph, starts, L: int, *, seed: int = 42, walk_id_base: int = 0,
                      out=None, steps=None, stream=None) -> torch.Tensor:
    """grape_walks_first_order.  steps: optional int64 tensor (device path: 1-element
    CUDA tensor, incremented on the device) to which realised transitions are added."""
    return _walks("grape_walks_first_order", g, starts, L, (), seed, walk_id_base, out, steps, stream)


def walks_node2vec(g: Graph, starts, L: int, p: float, q: float, *, seed: int = 42,
                   walk_id_base: int = 0, out=None, steps=None, stream=None) -> torch.Tensor:
    """grape_walks_node2vec (p = return, q = in-out parameter)."""
    return _walks("grape_walks_node2vec", g, starts, L, (float(p), float(q)), seed, walk_id_base,
                  out, steps, stream)


def walks_node2vec_cdf(g: Graph, starts, L: int, p: float, q: float, *, seed: int = 42,
                       walk_id_base: int = 0, out=None, steps=None, stream=None) -> torch.Tensor:
    """grape_walks_node2vec_cdf: node2vec with the paper's inverse-CDF sampler."""
    return _walks("grape_walks_node2vec_cdf", g, starts, L, (float(p), float(q)), seed, walk_id_base,
                  out, steps, stream)


def walks_node2vec_folded(g: Graph, starts, L: int, p: float, q: float, *, seed: int = 42,
                          walk_id_base: int = 0, out=None, steps=None, stream=None) -> torch.Tensor:
    """grape_walks_node2vec_folded: node2vec with outlier-folded rejection (same law, fewer
    attempts when p < min(1, q))."""
    return _walks("grape_walks_node2vec_folded", g, starts, L, (float(p), float(q)), seed, walk_id_base,
                  out, steps, stream)


def skipgram_pairs(g: Graph, walks, window: int, num_negatives: int, *, seed: int = 42, walk_id_base: int = 0,
                   out=None, stream=None):
    """grape_skipgram_pairs: SkipGram (center, context) pairs of every window offset and
    scale-free negatives.  walks: CUDA int32 [W, L] (a walk matrix).
    Returns (centers int32[S], contexts int32[S], negatives int32[S, K]), S = W*L*2*window;
    invalid slots hold PAD (-1)."""
    if not (torch.is_tensor(walks) and walks.is_cuda and walks.dim() == 2):
        raise ValueError("walks must be a 2-D CUDA tensor (a walk matrix)")
    if walks.dtype not in (torch.int32, torch.uint32):
        raise ValueError(f"walks must be int32 (u32 bit patterns), got {walks.dtype}")
    if walks.device.index != g.device:
        raise ValueError(f"walks on cuda:{walks.device.index}, graph on cuda:{g.device}")
    walks = walks.contiguous()
    W, L = walks.shape
    S = W * L * 2 * window
    with torch.cuda.device(g.device):
        if out is None:
            out = (torch.empty(S, dtype=torch.int32, device=walks.device),
                   torch.empty(S, dtype=torch.int32, device=walks.device),
                   torch.empty((S, num_negatives), dtype=torch.int32, device=walks.device))
        else:
            if len(out) != 3:
                raise ValueError("out must be (centers, contexts, negatives)")
            _check_out(out[0], (S,), str(g.device), "centers")
            _check_out(out[1], (S,), str(g.device), "contexts")
            _check_out(out[2], (S, num_negatives), str(g.device), "negatives")
        c, x, ng = out
        stream = _stream_handle(stream, g.device, (walks, c, x, ng))
        rc = _lib.grape_skipgram_pairs(g.handle, walks.data_ptr(), W, walk_id_base, L, window, num_negatives,
                                       seed, c.data_ptr(), x.data_ptr(), ng.data_ptr() if num_negatives else None,
                                       ctypes.c_void_p(stream))
    _capi.check(_lib, rc, "grape_skipgram_pairs")
    return c, x, ng


def walks_skipgram(g: Graph, starts, L: int, window: int, num_negatives: int, *, node2vec: bool = True,
                   p: float = 1.0, q: float = 1.0, seed: int = 42, pair_seed: int = 43, walk_id_base: int = 0,
                   out=None, steps=None, chunk_walks: int = 0, stream=None):
    """grape_walks_skipgram: the walks of walks_node2vec / walks_first_order streamed into
    skipgram_pairs without materialising the walk matrix (bit-identical to the two calls).
    starts: CUDA int32 [W].  Returns (centers int32[S], contexts int32[S], negatives
    int32[S, K]), S = W*L*2*window."""
    st = _as_tensor(starts, torch.int32)
    if not st.is_cuda or st.device.index != g.device:
        raise ValueError(f"starts must be a CUDA tensor on cuda:{g.device}")
    W = st.numel()
    S = W * L * 2 * window
    with torch.cuda.device(g.device):
        if out is None:
            out = (torch.empty(S, dtype=torch.int32, device=st.device),
                   torch.empty(S, dtype=torch.int32, device=st.device),
                   torch.empty((S, num_negatives), dtype=torch.int32, device=st.device))
        else:
            if len(out) != 3:
                raise ValueError("out must be (centers, contexts, negatives)")
            _check_out(out[0], (S,), str(g.device), "centers")
            _check_out(out[1], (S,), str(g.device), "contexts")
            _check_out(out[2], (S, num_negatives), str(g.device), "negatives")
        if steps is not None:
            _check_steps(steps, True, g.device)
        c, x, ng = out
        sh = _stream_handle(stream, g.device, (st, c, x, ng))
        rc = _lib.grape_walks_skipgram(g.handle, st.data_ptr(), W, walk_id_base, L, int(node2vec), float(p),
                                       float(q), seed, window, num_negatives, pair_seed, c.data_ptr(), x.data_ptr(),
                                       ng.data_ptr() if num_negatives else None,
                                       None if steps is None else steps.data_ptr(), int(chunk_walks),
                                       ctypes.c_void_p(sh))
    _capi.check(_lib, rc, "grape_walks_skipgram")
    return c, x, ng


def walks_approx(g: Graph, starts, L: int, degree_threshold: int, *, node2vec: bool = True, p: float = 1.0,
                 q: float = 1.0, seed: int = 42, walk_id_base: int = 0, out=None, steps=None,
                 stream=None) -> torch.Tensor:
    """grape_walks_approx: approximated walks with SUSS sub-sampling of rows with more than
    degree_threshold neighbours (Fig. 3)."""
    return _walks_approx(g, starts, L, int(node2vec), float(p), float(q), int(degree_threshold), seed,
                         walk_id_base, out, steps, stream)


def _walks_approx(g, starts, L, n2v, p, q, dT, seed, walk_id_base, out, steps, stream):
    st = _as_tensor(starts, torch.int32)
    W = st.numel()
    fn = _lib.grape_walks_approx
    dev = st.is_cuda
    if dev and st.device.index != g.device:
        raise ValueError(f"starts on cuda:{st.device.index}, graph on cuda:{g.device}")
    with torch.cuda.device(g.device):
        if out is None:
            out = (torch.empty((W, L), dtype=torch.int32, device=st.device) if dev else
                   torch.empty((W, L), dtype=torch.int32, pin_memory=True))
        else:
            _check_out(out, (W, L), str(g.device) if dev else "cpu", "out")
        if steps is not None:
            _check_steps(steps, dev, g.device)
        stream = _stream_handle(stream, g.device, (st, out) if dev else ())
        hs = ctypes.c_uint64(0)
        sp = (None if steps is None else steps.data_ptr()) if dev else ctypes.byref(hs)
        rc = fn(g.handle, st.data_ptr(), W, walk_id_base, L, n2v, p, q, dT, seed, out.data_ptr(), sp,
                ctypes.c_void_p(stream))
    _capi.check(_lib, rc, "grape_walks_approx")
    if not dev and steps is not None:
        steps += int(hs.value)
    return out


def walks_stats(g: Graph, starts, L: int, *, node2vec: bool, p: float = 1.0, q: float = 1.0,
                seed: int = 42, walk_id_base: int = 0, out=None, degree_threshold: int = 0,
                sampler: str = "rejection"):
    """grape_walks_stats: (walk matrix, dict of event counters) — diagnostics build of the
    same kernel (device buffers only; synchronous)."""
    st = _as_tensor(starts, torch.int32)
    if not st.is_cuda:
        raise ValueError("walks_stats needs device starts")
    if st.device.index != g.device:
        raise ValueError(f"starts on cuda:{st.device.index}, graph on cuda:{g.device}")
    W = st.numel()
    with torch.cuda.device(g.device):
        if out is None:
            out = torch.empty((W, L), dtype=torch.int32, device=st.device)
        else:
            _check_out(out, (W, L), str(g.device), "out")
        stats = _capi.WalkStats()
        smp = {"rejection": 0, "cdf": 1, "folded": 2}[sampler]
        rc = _lib.grape_walks_stats_ex(g.handle, st.data_ptr(), W, walk_id_base, L, int(node2vec),
                                       float(p), float(q), int(degree_threshold), smp, seed, out.data_ptr(),
                                       ctypes.byref(stats),
                                       ctypes.c_void_p(torch.cuda.current_stream(g.device).cuda_stream))
    _capi.check(_lib, rc, "grape_walks_stats_ex")
    return out, {f: int(getattr(stats, f)) for f in _capi.STATS_FIELDS}


# C-ABI names, for callers that mirror the header.
grape_graph_from_csr = graph_from_csr
grape_walks_first_order = walks_first_order
grape_walks_node2vec = walks_node2vec
grape_walks_stats = walks_stats
grape_walks_approx = walks_approx
grape_walks_node2vec_cdf = walks_node2vec_cdf
grape_walks_node2vec_folded = walks_node2vec_folded

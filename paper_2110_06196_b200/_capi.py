"""ctypes declarations of include/grape_walk.h (argument marshalling only).

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
as ``paper_2110_06196_b200/libgrape_walk.so``.  There is no fallback: if the
library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgrape_walk.so")

GRAPE_OK, GRAPE_EINVAL, GRAPE_ENOMEM, GRAPE_ECUDA = 0, 1, 2, 3
GRAPE_SYMMETRIC = 1 << 0
GRAPE_SKIP_VALIDATION = 1 << 1
GRAPE_NO_TABLES = 1 << 2
GRAPE_PAD = 0xFFFFFFFF

# Every entry point include/grape_walk.h declares (tests check the .so exports them all).
EXPORTS = (
    "grape_graph_from_csr", "grape_graph_from_csr_opts", "grape_graph_free", "grape_graph_get_info",
    "grape_walks_first_order", "grape_walks_node2vec", "grape_walks_approx", "grape_walks_node2vec_cdf", "grape_walks_node2vec_folded",
    "grape_skipgram_pairs", "grape_walks_skipgram", "grape_graph_partition",
    "grape_graph_dist_create", "grape_graph_dist_export", "grape_graph_dist_import", "grape_graph_dist_build",
    "grape_graph_dist_finish",
    "grape_walks_stats",
    "grape_walks_stats_ex",
    "grape_status_string", "grape_last_error", "grape_version",
)


class GraphInfo(ctypes.Structure):
    _fields_ = [
        ("num_nodes", ctypes.c_uint32),
        ("num_arcs", ctypes.c_uint64),
        ("weighted", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
        ("cw_bytes", ctypes.c_uint32),
        ("max_degree", ctypes.c_uint32),
        ("max_row_weight", ctypes.c_uint64),
        ("device_bytes", ctypes.c_uint64),
        ("device", ctypes.c_int),
        ("tables", ctypes.c_uint32),
        ("weights_symmetric", ctypes.c_uint32),
        ("table_bytes", ctypes.c_uint64),
        ("guide_factor", ctypes.c_uint32),
        ("guide_bytes", ctypes.c_uint32),
        ("record_bytes", ctypes.c_uint32),
        ("hash_h", ctypes.c_uint32),
        ("notri", ctypes.c_uint32),
        ("parts", ctypes.c_uint32),
        ("wide", ctypes.c_uint32),
    ]


class TableOptions(ctypes.Structure):
    _fields_ = [
        ("table_budget_bytes", ctypes.c_uint64),
        ("record_bytes", ctypes.c_uint32),
        ("guide_bytes", ctypes.c_uint32),
        ("guide_factor", ctypes.c_uint32),
        ("hash_h", ctypes.c_uint32),
    ]


class IpcHandle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 64)]


class PartExport(ctypes.Structure):
    _fields_ = [
        ("part", ctypes.c_uint32),
        ("device", ctypes.c_int),
        ("bytes", ctypes.c_uint64 * 4),
        ("handle", IpcHandle * 4),
    ]


STATS_FIELDS = ("sector_loads", "node_loads", "xnode_loads", "cw_probes", "col_probes", "col_loads",
                "attempts", "membership_tests", "start_loads", "steps", "guide_loads", "hash_probes",
                "alu_decisions", "iterations", "draw_iterations", "back_iterations")


class WalkStats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in STATS_FIELDS]


class GrapeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def load(path: str | None = None) -> ctypes.CDLL:
    # GRAPE_WALK_LIB: an alternative in-tree build of the same library (used by
    # tools/ experiments to compare compile-time variants); default LIB_PATH.
    path = path or os.environ.get("GRAPE_WALK_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA library first (`make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    vp, u32, u64, i32, dbl = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
    lib.grape_graph_from_csr.argtypes = [u32, u64, vp, vp, vp, i32, u32, ctypes.POINTER(vp)]
    lib.grape_graph_from_csr.restype = i32
    lib.grape_graph_from_csr_opts.argtypes = [u32, u64, vp, vp, vp, i32, u32, ctypes.POINTER(TableOptions),
                                              ctypes.POINTER(vp)]
    lib.grape_graph_from_csr_opts.restype = i32
    lib.grape_graph_free.argtypes = [vp]
    lib.grape_graph_free.restype = i32
    lib.grape_graph_get_info.argtypes = [vp, ctypes.POINTER(GraphInfo)]
    lib.grape_graph_get_info.restype = i32
    lib.grape_walks_first_order.argtypes = [vp, vp, u64, u64, u32, u64, vp, vp, vp]
    lib.grape_walks_first_order.restype = i32
    lib.grape_walks_node2vec.argtypes = [vp, vp, u64, u64, u32, dbl, dbl, u64, vp, vp, vp]
    lib.grape_walks_node2vec.restype = i32
    lib.grape_walks_approx.argtypes = [vp, vp, u64, u64, u32, i32, dbl, dbl, u32, u64, vp, vp, vp]
    lib.grape_walks_approx.restype = i32
    lib.grape_walks_node2vec_cdf.argtypes = [vp, vp, u64, u64, u32, dbl, dbl, u64, vp, vp, vp]
    lib.grape_walks_node2vec_cdf.restype = i32
    lib.grape_walks_node2vec_folded.argtypes = [vp, vp, u64, u64, u32, dbl, dbl, u64, vp, vp, vp]
    lib.grape_walks_node2vec_folded.restype = i32
    lib.grape_skipgram_pairs.argtypes = [vp, vp, u64, u64, u32, u32, u32, u64, vp, vp, vp, vp]
    lib.grape_skipgram_pairs.restype = i32
    lib.grape_walks_skipgram.argtypes = [vp, vp, u64, u64, u32, i32, dbl, dbl, u64, u32, u32, u64, vp, vp, vp, vp,
                                         u64, vp]
    lib.grape_walks_skipgram.restype = i32
    lib.grape_graph_partition.argtypes = [vp, u32, vp]
    lib.grape_graph_partition.restype = i32
    lib.grape_graph_dist_create.argtypes = [u32, u64, vp, vp, vp, i32, u32, ctypes.POINTER(TableOptions), u32, u32,
                                            ctypes.POINTER(vp)]
    lib.grape_graph_dist_create.restype = i32
    lib.grape_graph_dist_export.argtypes = [vp, ctypes.POINTER(PartExport)]
    lib.grape_graph_dist_export.restype = i32
    lib.grape_graph_dist_import.argtypes = [vp, ctypes.POINTER(PartExport)]
    lib.grape_graph_dist_import.restype = i32
    lib.grape_graph_dist_build.argtypes = [vp, u32, ctypes.POINTER(u32)]
    lib.grape_graph_dist_build.restype = i32
    lib.grape_graph_dist_finish.argtypes = [vp, u32]
    lib.grape_graph_dist_finish.restype = i32
    lib.grape_walks_stats.argtypes = [vp, vp, u64, u64, u32, i32, dbl, dbl, u64, vp,
                                      ctypes.POINTER(WalkStats), vp]
    lib.grape_walks_stats.restype = i32
    lib.grape_walks_stats_ex.argtypes = [vp, vp, u64, u64, u32, i32, dbl, dbl, u32, i32, u64, vp,
                                         ctypes.POINTER(WalkStats), vp]
    lib.grape_walks_stats_ex.restype = i32
    lib.grape_status_string.argtypes = [i32]
    lib.grape_status_string.restype = ctypes.c_char_p
    lib.grape_last_error.argtypes = []
    lib.grape_last_error.restype = ctypes.c_char_p
    lib.grape_version.argtypes = []
    lib.grape_version.restype = ctypes.c_char_p
    return lib


def check(lib: ctypes.CDLL, status: int, what: str) -> None:
    if status != GRAPE_OK:
        detail = lib.grape_last_error().decode(errors="replace")
        name = lib.grape_status_string(status).decode()
        raise GrapeError(status, f"{what}: {name}: {detail}")

"""Host-only checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/grape_walk.h declares, rejects bad arguments before touching
CUDA, and the product package never reaches the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "grape_walk.h")
PKG = os.path.join(ROOT, "paper_2110_06196_b200")
LIB = os.path.join(PKG, "libgrape_walk.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", ROOT, "-s", "paper_2110_06196_b200/libgrape_walk.so"])
    from paper_2110_06196_b200 import _capi
    return _capi.load(LIB)


def _declared():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(grape_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_abi():
    names = _declared()
    for must in ("grape_graph_from_csr", "grape_walks_first_order", "grape_walks_node2vec"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2110_06196_b200 import _capi
    names = _declared()
    assert sorted(_capi.EXPORTS) == names
    nm = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (grape_\w+)", nm))
    for n in names:
        assert n in exported, n
        assert hasattr(lib, n)


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(lib):
    assert lib.grape_status_string(0).decode() == "GRAPE_OK"
    assert "EINVAL" in lib.grape_status_string(1).decode()
    assert "sm_100a" in lib.grape_version().decode()


def test_argument_errors_before_any_cuda_call(lib):
    vp = ctypes.c_void_p
    fake = ctypes.create_string_buffer(256)          # stands in for a handle; never dereferenced
    buf = ctypes.create_string_buffer(64)
    # NULL graph / starts / out
    assert lib.grape_walks_node2vec(None, buf, 1, 0, 4, 1.0, 1.0, 42, buf, None, None) == 1
    assert lib.grape_walks_first_order(fake, None, 1, 0, 4, 42, buf, None, None) == 1
    assert b"non-NULL" in lib.grape_last_error()
    # L = 0
    assert lib.grape_walks_first_order(fake, buf, 1, 0, 0, 42, buf, None, None) == 1
    assert b"walk_length" in lib.grape_last_error()
    # bad p, q, ratio
    for p, q in [(0.0, 1.0), (-1.0, 2.0), (float("nan"), 1.0), (1.0, float("inf")), (2.0 ** 25, 1.0)]:
        assert lib.grape_walks_node2vec(fake, buf, 1, 0, 4, p, q, 42, buf, None, None) == 1
    # overflow of num_walks * L
    assert lib.grape_walks_first_order(fake, buf, 2 ** 62, 0, 8, 42, buf, None, None) == 1
    # SkipGram consumer: NULL graph / buffers, L = 0, window 0 / too large, slot-count overflow
    assert lib.grape_skipgram_pairs(None, buf, 1, 0, 4, 2, 1, 42, buf, buf, buf, None) == 1
    assert lib.grape_skipgram_pairs(fake, buf, 1, 0, 4, 2, 1, 42, buf, buf, None, None) == 1
    assert b"non-NULL" in lib.grape_last_error()
    assert lib.grape_skipgram_pairs(fake, buf, 1, 0, 4, 2, 0, 42, buf, buf, None, None) != 0   # K = 0: NULL negatives ok
    assert lib.grape_skipgram_pairs(fake, buf, 1, 0, 0, 2, 1, 42, buf, buf, buf, None) == 1
    assert lib.grape_skipgram_pairs(fake, buf, 1, 0, 4, 0, 1, 42, buf, buf, buf, None) == 1
    assert lib.grape_skipgram_pairs(fake, buf, 1, 0, 4, 1025, 1, 42, buf, buf, buf, None) == 1
    assert lib.grape_skipgram_pairs(fake, buf, 2 ** 58, 0, 64, 5, 5, 42, buf, buf, buf, None) == 1
    assert b"overflows" in lib.grape_last_error()
    assert lib.grape_skipgram_pairs(fake, buf, 4, 2 ** 64 - 2, 4, 2, 1, 42, buf, buf, buf, None) == 1   # wid wrap
    assert b"overflows" in lib.grape_last_error()
    # partition: NULL graph / devices, parts out of range
    devs = (ctypes.c_int * 2)(0, 0)
    assert lib.grape_graph_partition(None, 2, devs) == 1
    assert lib.grape_graph_partition(fake, 1, devs) == 1
    assert lib.grape_graph_partition(fake, 9, devs) == 1
    assert lib.grape_graph_partition(fake, 2, None) == 1
    # graph build: NULL out, NULL arrays, n = PAD, unknown flags
    h = vp()
    assert lib.grape_graph_from_csr(3, 0, buf, buf, None, 0, 0, None) == 1
    assert lib.grape_graph_from_csr(3, 2, None, buf, None, 0, 0, ctypes.byref(h)) == 1
    assert lib.grape_graph_from_csr(0xFFFFFFFF, 0, buf, buf, None, 0, 0, ctypes.byref(h)) == 1
    assert lib.grape_graph_from_csr(3, 0, buf, buf, None, 0, 1 << 7, ctypes.byref(h)) == 1
    assert h.value is None
    assert lib.grape_graph_free(None) == 0
    from paper_2110_06196_b200 import _capi
    info = _capi.GraphInfo()
    assert lib.grape_graph_get_info(None, ctypes.byref(info)) == 1


def test_product_never_touches_the_oracle():
    """The product package must not import, link or execute oracle/ (no CPU fallback)."""
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|grape_oracle|"
                                     r"\boracle_\w+\s*\(|pyoracle)", src), f
    mk = open(os.path.join(ROOT, "Makefile")).read()
    lib_rule = mk.split("$(LIB):")[1].split("\n\n")[0]
    assert "oracle" not in lib_rule


def test_binding_rejects_mismatched_output_buffers():
    """The binding checks caller-supplied outputs before handing their pointers to the
    library (shape, dtype, contiguity, memory kind): a wrong buffer is a ValueError, never
    a write past its end."""
    import torch
    import paper_2110_06196_b200 as grape
    ok = torch.empty((4, 5), dtype=torch.int32)
    grape._check_out(ok, (4, 5), "cpu", "out")
    grape._check_out(ok.view(torch.uint32), (4, 5), "cpu", "out")
    for bad, why in [(torch.empty((4, 4), dtype=torch.int32), "shape"),
                     (torch.empty((5, 4), dtype=torch.int32), "shape"),
                     (torch.empty((4, 5), dtype=torch.int64), "int32"),
                     (torch.empty((5, 4), dtype=torch.int32).t(), "contiguous"),
                     (torch.empty((4, 5, 1), dtype=torch.int32), "shape")]:
        with pytest.raises(ValueError, match=why):
            grape._check_out(bad, (4, 5), "cpu", "out")
    with pytest.raises(ValueError, match="cuda:0"):
        grape._check_out(ok, (4, 5), "0", "out")            # host tensor for a device call
    grape._check_steps(torch.zeros(1, dtype=torch.int64), False, 0)
    for bad in (torch.zeros(1, dtype=torch.int32), torch.zeros(2, dtype=torch.int64),
                torch.zeros((), dtype=torch.float64)):
        with pytest.raises(ValueError, match="int64"):
            grape._check_steps(bad, False, 0)
    with pytest.raises(ValueError, match="cuda:0"):
        grape._check_steps(torch.zeros(1, dtype=torch.int64), True, 0)


def test_chunked_table_layout_host_logic(tmp_path):
    """The chunk / owner arithmetic of the partitioned and distributed table layouts
    (csrc/internal.h), compiled for the host and checked exhaustively over sizes and
    owner counts (tests/pins/chunks_test.cpp)."""
    exe = tmp_path / "chunks_test"
    src = os.path.join(ROOT, "tests", "pins", "chunks_test.cpp")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I/usr/local/cuda/include", "-Iinclude", src, "-o", str(exe)],
                          cwd=ROOT)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and "chunks_test: ok" in out.stdout, out.stdout + out.stderr

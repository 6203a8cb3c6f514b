"""The bounds-checked build (libgrape_walk_checked.so, -DGRAPE_CHECKED=1).

compute-sanitizer is closed on the GPU pool ("runs under it have left GPUs needing a
reset"), so its memcheck / racecheck / initcheck role is filled by a build of the same
sources in which every table read (against the table's byte size), every arc / guide /
hash / node index a kernel derives (against the row or table it must lie in), every
walk-matrix write (s < L, x < n), every build-kernel table access (TabRef) and every
SkipGram negative (the row that holds arc e) is checked on the device; a failed check
prints the condition and traps, failing the call.  These tests run every device code
path through that build — each walk mode and table layout, the builders, the
partitioned and distributed tables, the SkipGram kernels, the host-buffer path — and
compare every result with the oracle.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2110_06196_b200", "libgrape_walk_checked.so")
pytestmark = pytest.mark.gpu


def _env():
    assert os.path.exists(LIB), "build the checked library first (make checked)"
    return dict(os.environ, GRAPE_WALK_LIB=LIB)


def test_every_device_path_under_the_checked_build():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], cwd=ROOT, env=_env(),
                       capture_output=True, text=True, timeout=1200)
    assert "GRAPE_CHECKED" not in p.stdout + p.stderr, (p.stdout + p.stderr)[-3000:]
    assert p.returncode == 0 and "all checks passed" in p.stdout, (p.stdout + p.stderr)[-3000:]


def test_distributed_tables_under_the_checked_build():
    p = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "tests/test_gpu_dist.py",
                        "-k", "cfg5 or tiny"], cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=1200)
    assert "GRAPE_CHECKED" not in p.stdout + p.stderr, (p.stdout + p.stderr)[-3000:]
    assert p.returncode == 0, (p.stdout + p.stderr)[-3000:]


def test_checked_library_is_loaded_by_the_binding():
    code = ("import paper_2110_06196_b200 as g, paper_2110_06196_b200._capi as c; "
            "import os; print(os.path.realpath(c.load()._name))")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=_env(), capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0 and p.stdout.strip().endswith("libgrape_walk_checked.so"), p.stdout + p.stderr

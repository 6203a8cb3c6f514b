"""bench.py's JSON-line contract (the driver parses it): the reference arm on CPU,
alone and under a world-size-2 torchrun (rank 0 alone prints, the other rank exits
0 without work); on the GPU, the product arm's line with every required key, at
N=1 and under torchrun with one NCCL rank."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config")


def _run(args, timeout=900, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    p = subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return [json.loads(ln) for ln in lines], p


def test_reference_arm_line():
    lines, _ = _run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "2",
                     "--warmup", "1", "--ref-budget", "0.3"])
    assert len(lines) == 1
    d = lines[0]
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "steps/s"
    assert d["config"]["workload"].startswith("BASELINE configs[0]")
    assert d["config"]["l2"].startswith("flushed")      # configs[0] fits in L2
    assert d["e2e"] == {"value": d["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]


def test_reference_arm_under_torchrun_prints_once():
    lines, _ = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                     "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--impl", "reference",
                     "--gpus", "2", "--config", "1", "--steps", "1", "--warmup", "0", "--ref-budget", "0.2"])
    assert len(lines) == 1 and lines[0]["impl"] == "reference"


@pytest.mark.gpu
def test_product_line_n1():
    lines, p = _run([sys.executable, "bench.py", "--config", "1", "--steps", "3", "--warmup", "3",
                     "--cpu-budget", "0.5"])
    assert len(lines) == 1
    d = lines[0]
    for k in REQUIRED + ("roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] >= 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    # DRAM traffic read from the GPU counters in this run (CUPTI, one untimed launch; configs[0]
    # is L2-resident, so only that it was measured is asserted).  On a box whose profiler an
    # earlier `ncu --set full` left unusable, CUPTI refuses the range (observed: Stop returns
    # CUPTI_ERROR_UNKNOWN in every later process until the box is recycled); bench.py then says
    # so on stderr and falls back to the committed capture, which it names
    if r["traffic_source"].startswith("measured in this run"):
        assert r["traffic"] > 0
        # ... and so are the issue counters of one more launch (the walker's other bound)
        iss = r["issue"]
        assert iss["warp_instructions_per_launch"] > 0 and 1 <= iss["active_threads_per_instruction"] <= 32
        assert 0 < iss["frac"] <= 1 and 0 < iss["issue_active_frac"] <= 1
        assert r["utilisation"]["highest"] in ("dram_traffic", "random_access", "issue")
    else:
        assert "dram probe: cupti" in p.stderr, p.stderr[-2000:]
        assert r["traffic_source"].startswith("profiles/traffic_cfg1.json") and r["traffic"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 4 * 10 ** 4 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_product_line_under_torchrun_one_rank():
    lines, _ = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                     "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "1",
                     "--config", "1", "--steps", "3", "--warmup", "3", "--no-cpu"])
    assert len(lines) == 1 and lines[0]["n_gpus"] == 1 and lines[0]["value"] > 0

"""bench.py's N > 1 rank path on real kernels.

Two ranks launched by torchrun run bench.py's own per-rank code — graph replica,
start-node slice [floor(r W/N), floor((r+1) W/N)) with walk_id_base = the slice
start, timed walk launches, max-over-ranks reduction — both on cuda:0 with the
gloo backend (NCCL refuses two ranks on one device; the walk kernels of the two
processes never wait on each other).  Each rank dumps its walk matrix; their
concatenation must equal the N = 1 run's matrix bit for bit, and a sample of rows
must equal the oracle's walks.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _bench(nproc, extra, port, tmp, tag):
    prefix = os.path.join(tmp, tag)
    if nproc == 1:
        cmd = [sys.executable, "bench.py"]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
               "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--device", "0",
               "--dist-backend", "gloo"]
    cmd += ["--gpus", str(nproc), "--steps", "3", "--warmup", "3", "--no-cpu", "--dump-walks", prefix] + extra
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stderr[-4000:]
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    parts = []
    for r in range(nproc):
        meta = json.load(open(f"{prefix}.rank{r}.json"))
        parts.append((meta["lo"], meta["hi"], np.load(f"{prefix}.rank{r}.npy"), meta["steps"]))
    return lines[0], parts


@pytest.mark.parametrize("cfg,extra", [(1, []), (2, ["--scale-down", "5", "--no-e2e"]),
                                       (5, ["--scale-down", "8", "--no-e2e"]),
                                       (2, ["--scale-down", "4", "--no-e2e", "--dist-tables", "--table-budget", "0.3"])],
                         ids=["cfg1", "cfg2-scaled", "cfg5-scaled", "cfg2-scaled-dist-tables"])
def test_two_ranks_strong_scaling_equals_one_rank(tmp_path, cfg, extra):
    """(last case: the tables built distributed over the two ranks, 0.3 GB each, bench
    --dist-tables; the N = 1 reference run builds them on one GPU)"""
    extra = ["--config", str(cfg)] + extra
    one_extra = [a for a in extra if a not in ("--dist-tables", "--table-budget", "0.3")]
    one, p1 = _bench(1, one_extra, 0, str(tmp_path), "n1")
    two, p2 = _bench(2, extra, 29600 + cfg + 10 * len(extra), str(tmp_path), "n2")
    if "--dist-tables" in extra:
        assert "distributed" in two["config"]["tables"] and "distributed over 2 GPUs" in two["metric"]
    assert one["scaling"] == two["scaling"] == "strong"
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    W = one["config"]["walks_total"]
    assert two["config"]["walks_total"] == W
    (lo1, hi1, full, steps1), = p1
    assert (lo1, hi1) == (0, W) and full.shape[0] == W
    # rank slices: contiguous, balanced, covering [0, W)
    p2 = sorted(p2, key=lambda t: t[0])
    assert p2[0][0] == 0 and p2[-1][1] == W and p2[0][1] == p2[1][0]
    assert abs((p2[0][1] - p2[0][0]) - (p2[1][1] - p2[1][0])) <= 1
    cat = np.concatenate([t[2] for t in p2])
    assert np.array_equal(cat, full)
    # the whole-job counters agree: realised steps per launch summed over ranks
    assert sum(t[3] for t in p2) == steps1
    assert len(two["rank_ms_per_step"]) == 2 and all(t > 0 for t in two["rank_ms_per_step"])
    assert two["value"] > 0 and one["value"] > 0
    # rows of rank 1's slice against the oracle, walk by walk (walk_id_base = slice start)
    from graphgen import config_graph, config_walks, starts_per_node
    from oracle.oracle import Oracle
    sd = int(extra[extra.index("--scale-down") + 1]) if "--scale-down" in extra else 0
    g = config_graph(cfg, scale_down=sd)
    wk = config_walks(cfg)
    starts = starts_per_node(g.n, wk["walks_per_node"]).numpy().view(np.uint32)
    o = Oracle(*g.numpy())
    lo, hi, mine, _ = p2[1]
    rng = np.random.default_rng(cfg)
    for i in np.unique(np.concatenate([rng.integers(lo, hi, 200), [lo, hi - 1]])):
        exp, _ = o.walks(starts[i:i + 1], wk["L"], mode=wk["mode"], p=wk["p"], q=wk["q"], seed=wk["seed"],
                         base=int(i))
        assert np.array_equal(mine[i - lo], exp[0]), int(i)

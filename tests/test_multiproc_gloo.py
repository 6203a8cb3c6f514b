"""Multi-process (world_size 2, gloo, CPU) checks of the N > 1 host logic:
sharding by walk id reproduces the single-process walk list bit for bit, and the
timing reduction takes the max over ranks / sum of steps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_06196_b200.shard import shard_range, weak_scaling_range, reduce_step_timing


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from graphgen import tiny_graph
        from oracle.oracle import Oracle
        g = tiny_graph(12, 80, 0.08, weighted=True)
        n, off, col, w = g.numpy()
        wpn = 3
        starts_all = np.tile(np.arange(n, dtype=np.uint32), wpn)          # iteration-major
        lo, hi = shard_range(len(starts_all), rank, world)
        mine, steps = Oracle(n, off, col, w).walks(starts_all[lo:hi], 20, p=0.5, q=2.0, seed=9, base=lo)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, mine, steps))
        t, s = reduce_step_timing(10.0 + rank, float(steps), world)
        q.put((rank, parts, t, s))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_partition():
    for total in (0, 1, 7, 10, 1000003):
        for world in (1, 2, 3, 8):
            rs = [shard_range(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    assert weak_scaling_range(100, 2, 4) == (200, 300)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_two_rank_gloo_sharding_is_bit_exact():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from graphgen import tiny_graph
    from oracle.oracle import Oracle
    g = tiny_graph(12, 80, 0.08, weighted=True)
    n, off, col, w = g.numpy()
    starts_all = np.tile(np.arange(n, dtype=np.uint32), 3)
    full, fsteps = Oracle(n, off, col, w).walks(starts_all, 20, p=0.5, q=2.0, seed=9)
    for rank, parts, t, s in res:
        cat = np.concatenate([m for (_, _, m, _) in sorted(parts, key=lambda x: x[0])])
        assert np.array_equal(cat, full)
        assert t == 11.0                      # max over ranks
        assert s == float(fsteps)             # sum of realised steps


def test_bench_rank_slices_strong_and_weak():
    """bench.py's N > 1 split: strong scaling shards the config's fixed
    iteration-major walk list into contiguous start-node slices (the union is the
    N = 1 list, each slice's walk_id_base is its start); weak scaling gives each rank
    its own block of the per-GPU workload."""
    import bench
    W = 10_000_000
    for world in (1, 2, 3, 4, 8):
        sl = [bench.rank_slice(W, W, r, world, "strong") for r in range(world)]
        assert sl[0][0] == 0 and sl[-1][1] == W
        assert all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
        assert sum(b - a for a, b in sl) == W
        wk = [bench.rank_slice(W, W, r, world, "weak") for r in range(world)]
        assert wk == [(r * W, (r + 1) * W) for r in range(world)]
    # one walk per node (configs 3-5): a rank's slice is a contiguous start-node range
    n = 1000
    starts = np.arange(n)
    for r in range(8):
        lo, hi = bench.rank_slice(n, n, r, 8, "strong")
        assert np.array_equal(starts[lo:hi], np.arange(lo, hi))

"""Two ranks on one GPU (gloo), distributed tables of configs[1] (tools):
each rank times its walk slice ALONE (the other waits at a barrier), then both together,
to separate same-device IPC access cost from two processes time-slicing one GPU."""
import os
import socket
import sys
import time

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, dist_tables, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2110_06196_b200 as grape
    from graphgen import config_graph, starts_per_node
    g = config_graph(2, device="cuda")
    if dist_tables:
        dg = grape.graph_from_csr_dist(g.off, g.col, g.w, device=0, symmetric=True,
                                       table_budget_bytes=int(24e9 / world))
    else:
        dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    g = g.to("cpu")
    torch.cuda.empty_cache()
    W = g.n * 10
    lo, hi = W * rank // world, W * (rank + 1) // world
    st = starts_per_node(g.n, 10, device="cuda")[lo:hi].contiguous()
    out = torch.empty((hi - lo, 80), dtype=torch.int32, device="cuda")
    res = {}

    def timed(k=3):
        grape.walks_node2vec(dg, st, 80, 0.5, 2.0, seed=42, walk_id_base=lo, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            grape.walks_node2vec(dg, st, 80, 0.5, 2.0, seed=42, walk_id_base=lo, out=out)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    for r in range(world):
        dist.barrier()
        if r == rank:
            res["alone_ms"] = timed()
        dist.barrier()
    dist.barrier()
    res["together_ms"] = timed()
    dist.barrier()
    res["info"] = {k: dg.info[k] for k in ("parts", "table_bytes", "guide_factor")}
    q.put((rank, res))
    dg.free()
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    modes = (True,) if len(sys.argv) > 2 else (False, True)
    for dist_tables in modes:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        ps = [ctx.Process(target=worker, args=(r, world, port, dist_tables, q)) for r in range(world)]
        for p in ps:
            p.start()
        out = sorted(q.get(timeout=900) for _ in range(world))
        for p in ps:
            p.join()
        print("dist_tables" if dist_tables else "replicated", out, flush=True)

"""Random 8-byte gathers from a local allocation vs the same-size allocation of another
process on the same GPU opened by CUDA IPC (torch.multiprocessing shares CUDA tensors that
way), in both processes.  Context for DESIGN.md §10b (distributed tables, ranks sharing a
device)."""
import time

import torch
import torch.multiprocessing as mp

N = 11 * (1 << 30) // 8   # 11 GiB of int64


def gather_ms(t, idx, k=5):
    t[idx].sum()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        s = t[idx].sum()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / k


def worker(rank, qs, out):
    torch.cuda.set_device(0)
    mine = torch.ones(N, dtype=torch.int64, device="cuda")
    qs[1 - rank].put(mine)           # shared by CUDA IPC
    other = qs[rank].get()
    idx = torch.randint(0, N, (1 << 26,), device="cuda")
    res = {"local_ms": gather_ms(mine, idx), "ipc_ms": gather_ms(other, idx)}
    out.put((rank, res))
    qs[rank].get()                   # keep tensors alive until both are done
    del other


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    qs = [ctx.Queue(), ctx.Queue()]
    out = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, qs, out)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(out.get(timeout=600) for _ in range(2))
    for q in qs:
        q.put(None)
    for p in ps:
        p.join(timeout=60)
    print(res)

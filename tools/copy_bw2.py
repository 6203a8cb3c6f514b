"""D2H bandwidth from pinned host memory with 1, 2 and 4 concurrent copy streams, and
D2H concurrent with a running kernel (context for the e2e host-buffer pipeline)."""
import time
import torch

n = 1 << 30   # 1 GiB per stream-chunk set
d = torch.empty(4 * n, dtype=torch.uint8, device="cuda")
h = torch.empty(4 * n, dtype=torch.uint8, pin_memory=True)
for k in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    per = (4 * n) // k
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                h[i * per:(i + 1) * per].copy_(d[i * per:(i + 1) * per], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"D2H 4 GiB over {k} stream(s): {4 * n / dt / 1e9:6.1f} GB/s")
# pageable vs pinned chunk sizes
for mb in (16, 64, 256):
    m = mb << 20
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range((4 * n) // m):
        h[i * m:(i + 1) * m].copy_(d[i * m:(i + 1) * m], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"D2H 4 GiB in {mb} MiB copies, one stream: {4 * n / dt / 1e9:6.1f} GB/s")

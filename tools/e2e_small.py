"""Per-call overhead of the host-buffer path on a small graph (configs[0])."""
import time, torch, sys
sys.path.insert(0, '.')
import paper_2110_06196_b200 as grape
from graphgen import config_graph, starts_per_node
g = config_graph(1)
dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
for W in (10000, 1000, 10):
    st = starts_per_node(g.n, 1)[:W].contiguous().pin_memory()
    out = torch.empty((W, 32), dtype=torch.int32, pin_memory=True)
    for k in range(3):
        t0 = time.perf_counter()
        grape.walks_first_order(dg, st, 32, seed=42, out=out)
        print("host W", W, k, round((time.perf_counter() - t0) * 1e3, 3), "ms", flush=True)
    dst = st.cuda(); dout = torch.empty((W, 32), dtype=torch.int32, device="cuda")
    for k in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        grape.walks_first_order(dg, dst, 32, seed=42, out=dout); torch.cuda.synchronize()
        print("dev  W", W, k, round((time.perf_counter() - t0) * 1e3, 3), "ms", flush=True)
for k in range(3):
    t0 = time.perf_counter(); s = torch.cuda.Stream(); torch.cuda.synchronize()
    print("stream", round((time.perf_counter() - t0) * 1e3, 3), "ms")

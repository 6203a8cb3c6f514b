import time, torch, sys
sys.path.insert(0, '.')
import paper_2110_06196_b200 as grape
from graphgen import config_graph, starts_per_node
g = config_graph(2, device="cuda")
dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
g = g.to("cpu"); torch.cuda.empty_cache()
W = g.n * 10
st = starts_per_node(g.n, 10).pin_memory()
out = torch.empty((W, 80), dtype=torch.int32, pin_memory=True)
for k in range(5):
    t0 = time.perf_counter()
    grape.walks_node2vec(dg, st, 80, 0.5, 2.0, seed=42, out=out)
    torch.cuda.synchronize()
    print("call", k, round((time.perf_counter() - t0) * 1e3, 1), "ms", flush=True)
dst = st.cuda(); dout = torch.empty((W, 80), dtype=torch.int32, device="cuda")
for k in range(3):
    t0 = time.perf_counter(); grape.walks_node2vec(dg, dst, 80, 0.5, 2.0, seed=42, out=dout); torch.cuda.synchronize()
    print("dev", k, round((time.perf_counter() - t0) * 1e3, 1), "ms")
    t0 = time.perf_counter(); out.copy_(dout); torch.cuda.synchronize(); print("copy", round((time.perf_counter() - t0) * 1e3, 1), "ms")

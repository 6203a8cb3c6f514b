"""Host-buffer (e2e) call of configs[1] vs staging chunk size (GRAPE_HOST_CHUNK_MB) for the
library in GRAPE_WALK_LIB (or the default): ms per call, and the plain D2H of the walk matrix.
Run under gpurun:  python tools/e2e_sweep.py 64 128 256 512"""
import os, subprocess, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] != "child":
    for mb in sys.argv[1:]:
        env = dict(os.environ, GRAPE_HOST_CHUNK_MB=mb)
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(f"chunk {mb:>5} MB: {r.stdout.strip()} {r.stderr.strip()[-300:] if r.returncode else ''}", flush=True)
    sys.exit(0)
import paper_2110_06196_b200 as grape
from graphgen import config_graph, starts_per_node
g = config_graph(2, device="cuda")
dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
g = g.to("cpu"); torch.cuda.empty_cache()
W = g.n * 10
st = starts_per_node(g.n, 10).pin_memory()
out = torch.empty((W, 80), dtype=torch.int32, pin_memory=True)
ts = []
for k in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    grape.walks_node2vec(dg, st, 80, 0.5, 2.0, seed=42, out=out)
    ts.append((time.perf_counter() - t0) * 1e3)
dout = torch.empty((W, 80), dtype=torch.int32, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); out.copy_(dout); torch.cuda.synchronize()
cp = (time.perf_counter() - t0) * 1e3
print(f"e2e ms {sorted(ts[2:])[1]:.1f} (min {min(ts[2:]):.1f})  plain D2H {cp:.1f} ms")

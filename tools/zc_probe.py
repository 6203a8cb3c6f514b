"""Host-buffer walks: staged chunks (default) vs the kernel writing rows straight into pinned
host memory (GRAPE_HOST_ZEROCOPY=1), configs[1]; outputs compared with the device call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_06196_b200 as grape
from bench import config_graph, _walk_recipe
from graphgen import starts_per_node

class A: config = 2; approx = 0; sampler = "rejection"; mode = None
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
A.config = cfg
wk = _walk_recipe(A)
g = config_graph(cfg, device=torch.device("cuda", 0))
dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric)
g = g.to("cpu"); torch.cuda.empty_cache()
W = min(g.n * wk["walks_per_node"], int(sys.argv[2]) if len(sys.argv) > 2 else 10**7)
L = wk["L"]
st_d = starts_per_node(g.n, wk["walks_per_node"], device="cuda")[:W].contiguous()
ref = grape.walks_node2vec(dg, st_d, L, wk["p"], wk["q"], seed=wk["seed"]) if wk["mode"] == "node2vec" else \
      grape.walks_first_order(dg, st_d, L, seed=wk["seed"])
torch.cuda.synchronize()
ref = ref.cpu()
h_st = st_d.cpu().pin_memory()
h_out = torch.empty((W, L), dtype=torch.int32, pin_memory=True)
def call():
    if wk["mode"] == "node2vec":
        grape.walks_node2vec(dg, h_st, L, wk["p"], wk["q"], seed=wk["seed"], out=h_out)
    else:
        grape.walks_first_order(dg, h_st, L, seed=wk["seed"], out=h_out)
for mode in ("staged", "zerocopy", "staged", "zerocopy"):
    if mode == "zerocopy":
        os.environ["GRAPE_HOST_ZEROCOPY"] = "1"
    else:
        os.environ.pop("GRAPE_HOST_ZEROCOPY", None)
    h_out.fill_(0)
    call(); call()
    ok = torch.equal(h_out, ref)
    ts = []
    for _ in range(5):
        t = time.perf_counter(); call(); ts.append(1e3 * (time.perf_counter() - t))
    print(f"config {cfg} {mode:9s} W={W} L={L}: equal to the device call: {ok}; ms per call {[round(x, 1) for x in ts]}", flush=True)

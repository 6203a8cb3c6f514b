"""Launch-time modes of the walk kernel on configs[1]: per graph build and per output
buffer, the mean of 3 timed launches (which allocation decides a slow run?)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2110_06196_b200 as grape
from graphgen import config_graph, config_walks, starts_per_node
wk = config_walks(2)
for trial in range(3):
    g = config_graph(2, device="cuda")
    torch.cuda.empty_cache()
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
    gc = g.to("cpu"); del g; torch.cuda.empty_cache()
    st = starts_per_node(gc.n, wk["walks_per_node"], device="cuda")
    for o in range(3):
        out = torch.empty((st.numel(), wk["L"]), dtype=torch.int32, device="cuda")
        for _ in range(2):
            grape.walks_node2vec(dg, st, wk["L"], wk["p"], wk["q"], seed=42, out=out)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize(); ev[0].record()
        for _ in range(3):
            grape.walks_node2vec(dg, st, wk["L"], wk["p"], wk["q"], seed=42, out=out)
        ev[1].record(); torch.cuda.synchronize()
        print(f"graph {trial} out {o} ptr {out.data_ptr():#x}: {ev[0].elapsed_time(ev[1]) / 3:.2f} ms", flush=True)
        del out
    dg.free(); del st; torch.cuda.empty_cache()

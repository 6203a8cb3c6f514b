"""Check tools/libgrape_dram_probe.so on a GPU: DRAM bytes of a torch kernel and of a walk call."""
import ctypes, os, sys
lib = ctypes.CDLL(os.path.join(os.getcwd(), "tools", "libgrape_dram_probe.so"))
lib.grape_dram_probe_error.restype = ctypes.c_char_p
print("init", lib.grape_dram_probe_init(), lib.grape_dram_probe_error(), flush=True)   # before any CUDA work
import torch
sys.path.insert(0, os.getcwd())
x = torch.ones(1 << 26, device="cuda")
torch.cuda.synchronize()
def probe(fn, name):
    rc = lib.grape_dram_probe_begin()
    print(name, "begin rc", rc, lib.grape_dram_probe_error())
    fn(); torch.cuda.synchronize()
    rd, wr, ns = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    rc = lib.grape_dram_probe_end(ctypes.byref(rd), ctypes.byref(wr), ctypes.byref(ns))
    print(name, "end rc", rc, lib.grape_dram_probe_error(), rd.value, wr.value, ns.value, flush=True)
probe(lambda: x.mul_(2.0), "torch mul (256 MB read + write)")
import paper_2110_06196_b200 as grape
from graphgen import config_graph
g = config_graph(2, scale_down=4, device="cuda")
dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True)
st = torch.arange(g.n, dtype=torch.int32, device="cuda")
grape.walks_node2vec(dg, st, 40, 0.5, 2.0); torch.cuda.synchronize()
probe(lambda: grape.walks_node2vec(dg, st, 40, 0.5, 2.0), "grape walk")

"""Beyond-BASELINE config 7 (past 2^32 arcs): build on the GPU, check the wide walker's
walks against the oracle on a sample, print the shape.  Run under gpurun."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2110_06196_b200 as grape  # noqa: E402
from graphgen import config_graph, config_walks  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

t0 = time.time()
g = config_graph(7, device="cuda")
print(f"generated n={g.n} m={g.m} ({g.m / 2**32:.3f} x 2^32) in {time.time() - t0:.0f} s", flush=True)
torch.cuda.empty_cache()
t0 = time.time()
# (past the automatic layout's 68 GB gather-reach cap: give the tables 100 GB)
dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=True, layout={"table_budget_bytes": int(100e9)})
torch.cuda.synchronize()
print(f"built in {time.time() - t0:.1f} s: {dg.info}", flush=True)
assert dg.info["tables"] == 1 and dg.info["wide"] == 1
deg = g.off[1:] - g.off[:-1]
hubs = torch.topk(deg, 20).indices
del deg
gc = g.to("cpu")
del g
torch.cuda.empty_cache()
wk = config_walks(7)
rng = np.random.default_rng(7)
sample = np.unique(np.concatenate([rng.integers(0, gc.n, 3000), hubs.cpu().numpy()])).astype(np.uint32)
st = torch.as_tensor(sample.view(np.int32)).cuda()
# walk ids = node ids (one walk per node, iteration-major): each sampled walk computed alone
out = torch.empty((len(sample), wk["L"]), dtype=torch.int32, device="cuda")
for i in range(len(sample)):   # walk_id_base = the node id, as in the full config run
    grape.walks_node2vec(dg, st[i:i + 1], wk["L"], wk["p"], wk["q"], seed=wk["seed"], walk_id_base=int(sample[i]),
                         out=out[i:i + 1])
torch.cuda.synchronize()
got = out.cpu().numpy().view(np.uint32)
o = Oracle(*gc.numpy())
bad = 0
for i, v in enumerate(sample):
    exp, _ = o.walks(sample[i:i + 1], wk["L"], mode="node2vec", p=wk["p"], q=wk["q"], seed=wk["seed"], base=int(v))
    bad += not np.array_equal(got[i], exp[0])
print(f"sampled walks: {len(sample)}, differing from the oracle: {bad}", flush=True)
dg.free()
sys.exit(1 if bad else 0)

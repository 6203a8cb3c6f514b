"""BASELINE.json configs[0..4] as (graph recipe, walk recipe) — DESIGN.md §5.

Graph seed = config number (1..5); walk seed = 42 everywhere (configs[0]
states 42, the others state none).  "cfgK" below is BASELINE.json configs[K-1].
"""
from __future__ import annotations

from .gen import chung_lu, rmat

CONFIGS = {
    1: dict(name="cfg1_chunglu_10k_first_order", graph=dict(kind="chung_lu", n=10_000, m=100_000, weights=None),
            mode="first_order", p=1.0, q=1.0, walks_per_node=1, L=32, seed=42),
    2: dict(name="cfg2_chunglu_1M_n2v_p0.5_q2", graph=dict(kind="chung_lu", n=1_000_000, m=20_000_000, weights=100),
            mode="node2vec", p=0.5, q=2.0, walks_per_node=10, L=80, seed=42),
    3: dict(name="cfg3_rmat24_n2v_p1_q0.25", graph=dict(kind="rmat", scale=24, ef=32, symmetric=True, weights=None),
            mode="node2vec", p=1.0, q=0.25, walks_per_node=1, L=100, seed=42),
    4: dict(name="cfg4_chunglu_50M_n2v_p2_q0.5", graph=dict(kind="chung_lu", n=50_000_000, m=1_000_000_000, weights=1000),
            mode="node2vec", p=2.0, q=0.5, walks_per_node=1, L=100, seed=42),
    5: dict(name="cfg5_rmat26_directed_n2v_p0.25_q4", graph=dict(kind="rmat", scale=26, ef=16, symmetric=False,
                                                                weights=("geometric", 10.0), sinks=0.05),
            mode="node2vec", p=0.25, q=4.0, walks_per_node=2, L=64, seed=42),
    # beyond BASELINE (not a BASELINE config): configs[3]'s recipe at 2.2e9 arcs, past the 2^31-arc
    # range the round-1 tables stopped at (index ranges); bench.py --config 6
    6: dict(name="x6_chunglu_55M_2.2Garcs_n2v_p2_q0.5", graph=dict(kind="chung_lu", n=55_000_000, m=1_110_000_000,
                                                                  weights=1000),
            mode="node2vec", p=2.0, q=0.5, walks_per_node=1, L=100, seed=42),
    # beyond BASELINE: past 2^32 arcs (the wide walker): unweighted Chung-Lu with
    # 100M nodes and 2.4e9 edge draws -> ~4.7e9 arcs; bench.py --config 7 --max-walks 20000000
    7: dict(name="x7_chunglu_100M_4.7Garcs_n2v_p2_q0.5", graph=dict(kind="chung_lu", n=100_000_000,
                                                                   m=2_400_000_000, weights=None),
            mode="node2vec", p=2.0, q=0.5, walks_per_node=1, L=100, seed=42),
}


def config_graph(k: int, device="cpu", *, scale_down: int = 0):
    """Build configs[k-1]'s graph.  scale_down > 0 shrinks it (n >> scale_down,
    m >> scale_down) for quick tests; 0 is the full BASELINE size."""
    g = CONFIGS[k]["graph"]
    if g["kind"] == "chung_lu":
        n, m = g["n"] >> scale_down, g["m"] >> scale_down
        return chung_lu(n, m, seed=k, weights=g["weights"], device=device,
                        name=CONFIGS[k]["name"] + (f"/2^{scale_down}" if scale_down else ""))
    return rmat(g["scale"] - scale_down, g["ef"], seed=k, symmetric=g["symmetric"],
                weights=g["weights"], device=device, sink_fraction=g.get("sinks"),
                name=CONFIGS[k]["name"] + (f"/2^{scale_down}" if scale_down else ""))


def config_walks(k: int):
    c = CONFIGS[k]
    return dict(mode=c["mode"], p=c["p"], q=c["q"], walks_per_node=c["walks_per_node"], L=c["L"],
                seed=c["seed"])

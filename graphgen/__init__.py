"""Seeded synthetic graph generators — shared INPUT module (no walk arithmetic).

Both the oracle side (tests) and the CUDA side (tests, bench) take their
graphs from here; nothing in this package draws a walk, computes a prefix sum
or a threshold.  Generators are counter-based (splitmix64 of (seed, stream,
index)) and use only integer ops plus correctly-rounded IEEE double
add/multiply, and a stable sort; so the same call gives bit-identical CSR
arrays on CPU and on CUDA (tests/test_graphgen.py, tests/test_gpu_graphgen.py).

The recipes are DESIGN.md §5 ("input recipe"), following SURVEY.md §8(d):
the paper's real graphs (Fig.2's 44 graphs, sk-2005 P:118/P:288, STRING
PPI P:110) are not available, so these stand in for them with the shapes
BASELINE.json names.
"""
from .gen import (  # noqa: F401
    CSR,
    splitmix64,
    chung_lu,
    rmat,
    tiny_graph,
    csr_from_arcs,
    starts_per_node,
)
from .configs import CONFIGS, config_graph, config_walks  # noqa: F401

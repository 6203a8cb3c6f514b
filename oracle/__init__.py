"""CPU oracle for the GRAPE walk hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2110_06196_b200`` never imports it (a test checks).

* ``grape_oracle.c`` — the oracle proper: plain single-threaded C, built into
  ``liboracle.so`` and called through ``ctypes`` by :mod:`oracle.oracle`.
* ``pyoracle.py`` — a pure-Python transliteration (Python big integers) used
  on tiny graphs to cross-check the C code bit for bit.

Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n, §8(c) =
SURVEY.md §8(c) readings (restated in DESIGN.md §3).
"""
from .oracle import (  # noqa: F401
    PAD,
    Oracle,
    build_oracle,
    draw,
    bounded,
    thresholds,
    prefix,
    upper_bound,
    walks,
    first_order_steps,
    node2vec_steps,
    philox4x32_10,
    suss,
)

"""The oracle: a plain, slow, double-precision CPU implementation of the Tiny-Twin
hot path (arXiv 2601.08217). TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. It shares no code with
``paper_2601_08217_b200`` (the CUDA path) and imports nothing from it; both sides
take their seeded inputs from ``ttsynth`` only.

See ``oracle/tt_oracle.c`` for the definition and its citations, and DESIGN.md §3
for the readings of the paper it follows.
"""
from .oracle import (  # noqa: F401
    build,
    lib,
    philox4x32_10,
    noise_scale,
    noise_block,
    normal_pair,
    radius_all,
    angle_all,
    convolve,
    convolve_points,
    aggregate,
    select_top_n,
    synth_jakes,
    OracleError,
)

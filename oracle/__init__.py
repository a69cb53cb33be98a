"""CPU fp64 ORACLE for CP-ALS / CP-ALS-QR / CP-ALS-QR-SVD (arXiv 2112.10855).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
cpu_baseline / `--impl reference` legs may import, call or execute anything under
`oracle/`.  The product path (`paper_2112_10855_b200`, `libcpqr.so`) never imports it and
shares no code with it; the only shared module is the seeded input generator
`paper_2112_10855_b200/synth.py`, which holds none of the method's arithmetic.

Every function cites the PAPER.md passage (line numbers of /root/reference/PAPER.md,
section / equation / algorithm line) it restates.  Where the paper is silent, the reading
taken is the one listed in SURVEY.md §8(c) and DESIGN.md §Readings, cited as "reading k".

Pins: see tests/test_oracle_pins.py.  All functions here are pinned; none is
"parity unpinned" except the paper's absent figures (not implemented here).
"""
from .cp_oracle import *  # noqa: F401,F403

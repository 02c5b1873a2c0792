"""AutoScout scoring ORACLE — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct CPU definition of the hot path that the
CUDA library (`paper_2603_11603_b200`) must reproduce: decode a candidate index of the
hierarchical configuration space, apply conditional validity, run the analytical
iteration-time/memory simulator, evaluate the GP posterior and the acquisition, keep a top-k.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything under ``oracle/``.  The product
path never routes through it, and it shares no code with the CUDA path: it parses the
space JSON itself, enumerates configurations by its own memoised dynamic program (not the
library's structure tables), solves the GP by a dense direct solve (not Cholesky/L^-1) and
scores in FP64.

Citations: ``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n,
``SURVEY §x`` = /root/repo/SURVEY.md.  Every reading of an ambiguous passage is listed in
DESIGN.md §3 ("Readings").

Modules
  space    load/validate the space JSON, activity (G1), constraints (G2/G3), CVI DP
  sim      analytical simulators (SPEC mode, derived mode, serving) + FP64 resource mask (G4)
  gp       feature map, Matern-5/2 kernel, GP fit by dense solve, posterior
  acq      EI (as log EI), LCB, SIM scores
  feistel  splitmix64 + 4-round Feistel permutation used by SAMPLE mode
  run      score a batch (RANGE / SAMPLE), per-candidate records, exact top-k

Pinning status (see tests/test_oracle_*.py): every module is pinned by values or properties
that do not come from this package (SPEC/PAPER examples, closed forms, mpmath/quad
integration, brute-force enumeration, Schur-complement identities).  The serving simulator
(sim.serve) is pinned only by hand-evaluated special cases and monotonicity: the paper
has no serving model (SURVEY §8(c) ledger #3) -- "parity partially unpinned" for its
non-special-case values, as stated in DESIGN.md.
"""

from . import space, sim, gp, acq, feistel, ensemble, run  # noqa: F401

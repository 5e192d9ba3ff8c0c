"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what FastFourierSAT's hot path
computes (PAPER.md arXiv 2308.15020), written from the paper and pinned by
tests/test_oracle_pins.py against values the paper prints, closed forms and brute force.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import, call, link or execute anything in this package.  The product path
(paper_2308_15020_b200/) never does: it fails loudly when its CUDA library is missing.

Tiers:
  T0 exact.py   exact rationals: Thm. 1 Walsh coefficients, ESPs (Eq. 6), WE = f^.esp (Eq. 3)
  T1 exact.py   brute-force multilinear extension over all 2^k corners (k <= 16)
  T2 dp.c       fp64 GradSAT/BDD probability DP (Alg. 5) for f, grad f, checks
     solve.py   Alg. 1 / Alg. 4 / Prop. 3 / rephasing semantics on top of T2
     philox.py  Philox4x32-10 from its published definition
Parity status: every function is pinned (no "parity unpinned" entries).
"""

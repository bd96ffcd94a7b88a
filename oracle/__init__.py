"""CPU FP64 oracle for the GMT matrix-free GMG hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import,
call or execute anything under ``oracle/``.  The product path
(``paper_2604_26518_b200`` + ``libgmt``) never imports it, and this package
never imports the product: the two share no code.  The only shared module is
``synth`` (seeded input generators, none of the method's arithmetic).

Everything here is written for a reader checking it against PAPER.md by eye:
plain definitions, fp64, global sparse matrices (scipy.sparse as the
library primitive), no blocking/fusion/reordering beyond what the paper's
definition or algorithm states.  Each function cites the passage it follows.

Modules
  fem      -- element matrices (App. F1/F2), EBE operator (Sec. 4.6 Eq. 14),
              global assembly K and load vector f (Eq. 3), C^H (App. F1/F2)
  transfer -- trilinear prolongation P and R = P^T (App. E1/E2)
  gmg      -- Galerkin coarse operators (Sec. 3.2 "Operator Consistency",
              Sec. 4.6 Eq. 17), damped-Jacobi smoothing (Sec. 4.6 Eq. 16 with
              the north-star smoother), V-cycle (Alg. 1 / Alg. 2), solve loop

Parity pins: see tests/test_oracle_*.py.  Every function listed above is
pinned by at least one independent check (closed forms, invariants, brute
force or a dense direct solve).  No function here is "parity unpinned".
"""

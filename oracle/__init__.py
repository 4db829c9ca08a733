"""CPU oracle for arXiv 1909.10616 (G-BFS / N-A2C GEMM-tiling tuners).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_1909_10616_b200``) never imports it and shares no code, header,
table or constant generator with it.

Citation convention: ``P:n`` is line n of the paper's PAPER.md, ``S:n`` line n
of SPEC.md; section / equation / algorithm labels are given alongside.
Readings of passages the paper leaves open are listed in DESIGN.md §3
("Readings") under the labels Z1..Z23 used below.

Modules
  space    -- Eq. 1-9 configuration space: count, enumerate, rank, J, step, g(s)
  hw       -- J_hw: the per-family launch limits (P:191 footnote), DESIGN.md §4
  rng      -- SplitMix64 stream + sampling (reading Z5, O7)
  costs    -- deterministic cost tables T1 and T2 ("randomly
              generated reward function")
  gbfs     -- Algorithm 1
  mlp      -- the actor / critic networks of Algorithm 2
  na2c     -- Algorithm 2
  measure  -- cost aggregation over repeated trials (reading Z10)
  gemm     -- C = A.B in double and in sequential-k fp32 fmaf (P:113, P:125,
              P:166); the arithmetic lives in gemm_ref.c

Parity status: every function is pinned by ``tests/test_oracle_*.py``.  The
N-A2C networks sum in a fixed order with C-library transcendentals (reading
Z24), so library trajectories are compared exactly at every eps.
"""

"""CPU oracle for the Paralpha Richardson iteration — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct numpy (fp64 / complex128) implementation of what
one alpha-circulant preconditioned Richardson iteration computes
(§2), written from the paper.  It shares no code with the
CUDA path (paper_2103_12571_b200/): neither imports the other.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import it.  The product path never routes through it.

Modules
  collocation  Radau IIA nodes and Q
  operators    periodic centred-FD operators A and their Fourier symbols
  schedule     Algorithm 2's alpha/m_k recurrence
  paralpha     the iteration u <- u + C_alpha^{-1}(w - C u) in three tiers
               (dense LU / spatial-Fourier / per-mode), brute force, sequential
               Radau IIA stepping, single-mode closed form

Parity pins: every function is pinned in tests/test_oracle_*.py against values
the paper prints, closed forms, invariants or brute force.
"""

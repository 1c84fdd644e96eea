"""TQSim CPU oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct numpy (complex128) implementation of what the
TQSim hot path computes (arXiv 2203.13892; citations are PAPER.md lines "P:n"
with their section/equation, and SPEC.md lines "S:n"; SURVEY.md §8(c) holds the
readings of ambiguous passages, repeated in DESIGN.md).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything in this package.  The
product (`paper_2203_13892_b200/`) never imports it, and this package never
imports the product: the two share no code, tables or constants; only the
seeded input generators in `workloads/` serve both.

Modules
  philox       Philox4x32-10 counter-based RNG (Salmon et al. 2011), pure ints + numpy
  gates        gate matrices and the lowering of CP / SWAP
  statevector  apply gates to a 2^n complex128 vector (little endian)
  noise        keyed depolarizing draws (§2.5, Eq.3 context)
  planner      DCP (§3.2, Eqs. 3-5), fixed arities, tree counts (Eq.2)
  tree         tree simulation with reuse (§3.1), per-leaf flat
               recompute, leaf sampling (§2.3) and readout
  density      density-matrix evolution (Eq.1) for brute-force pins on 2-4 qubits
  metrics      fidelity / normalized fidelity (Eqs. 6-7)

Parity status: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py; see DESIGN.md "Oracle pins".  Nothing is "parity unpinned"
except what DESIGN.md lists.
"""

"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy / scipy / plain C,
float64 / complex128) of what the CUDA path computes, written from PAPER.md
(arXiv:1411.4356).  Every function cites the passage it follows as
``PAPER.md:<line> (<section / equation>)``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import, call, link or execute anything in here.
The product package ``paper_1411_4356_b200`` never imports it, and this package
never imports the product: the two share no code (only ``workloads.py``, which
holds parameter sets and seeded random generators, no arithmetic of the method).

Modules
  liouvillian  Eq. (1) Hamiltonian, Eq. (3) Lindblad superoperator (column
               stacking, Eq. (4)), Eq. (5) trace-constrained system.
  superop_dense  an independent dense construction of the same superoperator
               (applies Eq. (3) to every basis matrix) -- used only as a pin.
  metrics      sec. II bandwidth / profile.
  rcm          sec. III reverse Cuthill-McKee (Python); rcm_ref.c is a second,
               independent C implementation of the same rule.
  ilut         sec. II dual-threshold incomplete LU (plain C in ilut.c).
  trisolve     forward / backward substitution with the ILUT factors.
  gmres        sec. IV restarted GMRES(m) with left preconditioning, Eq. (8).
  steadystate  the end-to-end oracle driver, the direct solve of Eq. (5), and
               the observables <a^+a>, <b^+b>.
"""

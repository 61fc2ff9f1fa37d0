"""CPU oracle for the VoxCap Galerkin system -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct reference for what the CUDA path computes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference`` leg may
import it; the product package ``paper_2004_02609_b200`` never does, and the two share no
code (only the input generators in ``voxgen/``, which hold none of the method's arithmetic).

What it computes, each function citing the passage it follows:
  enumerate_panels  -- voxel faces -> conductor / dielectric panels
  kappa             -- panel-pair integrals, binary128 closed forms (App. A)
  assemble          -- dense A = [0; I] + [P; E] (Eq. 4; Eqs. 5-7)
  matvec            -- y = A x (Eq. 4)
  solve_capacitance -- unit-potential solves and C = V^T rho_c with free-charge scaling
                       (Eq. 8)
  precond_apply     -- block-diagonal-diagonal preconditioner (Eq. 14)

Pins (tests/test_oracle_*.py): textbook self term, brute-force quadrature, symbolic
antiderivative checks, Gauss's law, cube/sphere physics, Maxwell invariants.  No function is
"parity unpinned".
"""
from .voxcap_oracle import *  # noqa: F401,F403
from .voxcap_oracle import __all__  # noqa: F401

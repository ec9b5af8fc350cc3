"""B200-native per-stage graph update of the convex-limited IDP Q1 Euler scheme.

Drop-in for the reference's `eulerflow.Solver` hot path (arXiv 2007.00094,
/root/reference/pkg/src/eulerflow/stepper.py).  The compute path is the
sm_100a library libef_b200.so (csrc/), bound through the C-ABI in
include/ef_b200.h; there is no CPU fallback.
"""

from .physics import AIR, AdmissibilityError, GasConstants
from .problems import BoundaryConditions, PrecomputedMatrices
from .stepper import STEP_NAMES, Solver, compute_tau, shared_pow

__all__ = ["Solver", "BoundaryConditions", "PrecomputedMatrices", "compute_tau", "GasConstants", "AIR",
           "AdmissibilityError", "STEP_NAMES", "shared_pow"]

"""Gas constants and admissibility, mirroring the reference's physics module.

`GasConstants` computes its derived constants in fp64 exactly as
`/root/reference/pkg/src/eulerflow/physics.py:33-52` does, so the values the
kernels receive are bit-identical to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["GasConstants", "AIR", "AdmissibilityError", "internal_energy", "is_admissible", "pressure",
           "n_variables"]


@dataclass(frozen=True)
class GasConstants:
    gamma: float = 7.0 / 5.0
    gm1: float = field(init=False)
    gp1_inv: float = field(init=False)
    gm1_over_2g: float = field(init=False)
    two_g_over_gm1: float = field(init=False)

    def __post_init__(self):
        if not self.gamma > 1.0:
            raise ValueError(f"gamma must exceed 1, got {self.gamma}")
        object.__setattr__(self, "gm1", self.gamma - 1.0)
        object.__setattr__(self, "gp1_inv", 1.0 / (self.gamma + 1.0))
        object.__setattr__(self, "gm1_over_2g", (self.gamma - 1.0) / (2.0 * self.gamma))
        object.__setattr__(self, "two_g_over_gm1", 2.0 * self.gamma / (self.gamma - 1.0))


AIR = GasConstants()


class AdmissibilityError(ValueError):
    """Raised when a state violates rho > 0 or internal energy > 0 (physics.py:55-56)."""


def n_variables(dim: int) -> int:
    return dim + 2


def internal_energy(U: np.ndarray) -> np.ndarray:
    return U[..., -1] - 0.5 * (U[..., 1:-1] * U[..., 1:-1]).sum(axis=-1) / U[..., 0]


def is_admissible(U: np.ndarray) -> np.ndarray:
    return (U[..., 0] > 0.0) & (internal_energy(U) > 0.0)


def pressure(U: np.ndarray, gas: GasConstants = AIR) -> np.ndarray:
    """p = (gamma - 1) eps (physics.py:92-94)."""
    return gas.gm1 * internal_energy(U)

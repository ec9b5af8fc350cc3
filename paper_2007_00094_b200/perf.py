"""Algorithmic memory traffic of one forward-Euler stage.

Restates the reference's roofline model `perf.predict_traffic`
(/root/reference/pkg/src/eulerflow/perf.py:47-89; paper Table 3,
PAPER.md:1761-1791) in doubles per stencil nonzero per phase.  Its counting
rules (perf.py:3-13): 4-byte column indices = 0.5 doubles/nnz; streamed
per-nnz matrices read once; per-node arrays cost size / average cardinality;
transposed gathers are free; per-node stores add a read-for-ownership.

These figures are the ALGORITHMIC bytes of the roofline fraction reported by
bench.py; the kernels here move fewer bytes than the model
because P_ij is rebuilt in registers instead of being stored and re-read, so
ncu's dram bytes are reported next to it.
"""

from __future__ import annotations

from typing import Dict

__all__ = ["predict_traffic", "stage_doubles_per_nnz", "KERNEL_OF_PHASE", "PHASES"]

INDEX_COST = 0.5
PHASES = ["step0", "step1", "step2", "step3", "step4", "step5", "step6"]
# phase -> the kernel(s) of libef_b200.so that implement it; step5 (one per
# extra limiter pass) is two kernels, the row update of the previous pass and
# the edge limiter of the next one
KERNEL_OF_PHASE = {
    "step0": "k_final (fused nodal update)",
    "step1": "k_edge_visc",
    "step2": "k_row_visc",
    "step3": "k_low_order",
    "step4": "k_edge_lim",
    "step5": "k_row_upd + k_edge_lim",
    "step6": "k_final",
}


def predict_traffic(dim: int, card: int) -> Dict[str, float]:
    """Doubles per nnz (reads + writes + rfo) per phase, perf.py:47-89."""
    nvar = dim + 2
    c = float(card)
    upper = (c + 1) / (2 * c)
    t = {
        "step0": (nvar / c) + (2 / c) + (2 / c),
        "step1": (dim + 1 + INDEX_COST + (nvar + 1) / c) + (upper + 1 / c) + (1 / c),
        "step2": (upper + 1 + 6 / c) + ((c - 1) / (2 * c)) + 0.0,
        "step3": (2 + dim + INDEX_COST + (2 * nvar) / c) + ((2 * nvar + 3) / c) + ((2 * nvar + 3) / c),
        "step4": (2 + INDEX_COST + (3 * nvar + 5) / c) + float(nvar + 1) + 0.0,
        "step5": (nvar + 1 + INDEX_COST + (nvar + 3) / c) + (1 + nvar / c) + (nvar / c),
        "step6": (nvar + 1 + INDEX_COST + nvar / c) + (nvar / c) + (nvar / c),
    }
    return t


def stage_doubles_per_nnz(dim: int, card: int, passes: int = 2) -> float:
    """Whole-stage model: step5 counted once per non-final pass (passes >= 1)."""
    t = predict_traffic(dim, card)
    total = t["step0"] + t["step1"] + t["step2"] + t["step3"]
    if passes > 0:
        total += t["step4"] + (passes - 1) * t["step5"] + t["step6"]
    return total

"""Algorithmic memory traffic of one forward-Euler stage.

Restates the reference's roofline model `perf.predict_traffic`
(/root/reference/pkg/src/eulerflow/perf.py:47-89; paper Table 3,
PAPER.md:1761-1791) in doubles per stencil nonzero per phase.  Its counting
rules (perf.py:3-13): 4-byte column indices = 0.5 doubles/nnz; streamed
per-nnz matrices read once; per-node arrays cost size / average cardinality;
transposed gathers are free; per-node stores add a read-for-ownership.

These figures are the ALGORITHMIC bytes of the roofline fraction reported by
bench.py.  The kernels move a different number of bytes
(L2 absorbs the neighbour re-reads; P and min(l) are stored per slot), so the
report puts ncu's measured DRAM bytes per launch next to the model when a
capture is available (profiles/ncu_traffic.json).

`format_table`, `write_csv` and `report` keep the reference's report API
(perf.py:92-153) with measured seconds per phase from `Solver.timers`.
"""

from __future__ import annotations

import csv
import json
import os
from typing import Dict, Optional

__all__ = ["predict_traffic", "stage_doubles_per_nnz", "KERNEL_OF_PHASE", "PHASES", "format_table",
           "write_csv", "report"]

DEFAULT_CARD = {2: 9, 3: 27}
_NCU = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    "ncu_traffic.json")

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


def _measured(solver) -> Dict[str, float]:
    if solver is None or solver.n_euler_steps == 0:
        return {}
    return {k: v / solver.n_euler_steps for k, v in solver.timers.items()}


def _ncu_bytes(config: Optional[str]) -> Dict[str, float]:
    """DRAM bytes per launch of each phase's kernel(s) from a committed capture."""
    if not config or not os.path.exists(_NCU):
        return {}
    with open(_NCU) as fh:
        k = json.load(fh).get(config, {})
    out = {}
    for ph, name in KERNEL_OF_PHASE.items():
        if ph == "step5":
            parts = [k.get("k_row_upd"), k.get("k_edge_lim#2")]
        else:
            parts = [k.get(name)]
        if all(parts):
            out[ph] = sum(p["traffic_bytes"] for p in parts)
    return out


def format_table(dim: int, card: Optional[int] = None, solver=None, config: Optional[str] = None) -> str:
    """Model table in doubles per nonzero; with a solver that has stepped, the
    measured seconds per stage and the achieved GB/s by the model; with a
    config name, ncu's measured DRAM bytes per launch."""
    card = DEFAULT_CARD[dim] if card is None else card
    pred = predict_traffic(dim, card)
    meas = _measured(solver)
    ncu = _ncu_bytes(config)
    nnz = getattr(solver, "nnz_owned", None)
    head = f"{'phase':8} {'dbl/nnz':>8} {'kernel':26}"
    if meas:
        head += f" {'s/stage':>11} {'model GB/s':>11}"
    if ncu:
        head += f" {'ncu MB':>9}"
    lines = [f"memory traffic model, dim={dim}, stencil cardinality={card} (doubles per nonzero)", head]
    for ph in PHASES:
        row = f"{ph:8} {pred[ph]:8.3f} {KERNEL_OF_PHASE[ph][:26]:26}"
        if meas:
            t = meas.get(ph, 0.0)
            gbs = (8.0 * pred[ph] * nnz / t / 1e9) if (t > 0 and nnz) else 0.0
            row += f" {t:11.3e} {gbs:11.1f}"
        if ncu:
            row += f" {ncu[ph] / 1e6:9.1f}" if ph in ncu else f" {'':>9}"
        lines.append(row)
    if solver is not None:
        lines.append(f"syncs={solver.comm.sync_count} volume={solver.comm.sync_volume} doubles "
                     f"over {solver.n_euler_steps} substeps")
    return "\n".join(lines)


def write_csv(path: str, dim: int, card: Optional[int] = None, solver=None) -> None:
    """The model (and measured seconds per stage when available) as CSV."""
    card = DEFAULT_CARD[dim] if card is None else card
    pred = predict_traffic(dim, card)
    meas = _measured(solver)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["phase", "kernel", "total_per_nnz", "measured_seconds_per_substep"])
        for ph in PHASES:
            w.writerow([ph, KERNEL_OF_PHASE[ph], f"{pred[ph]:.6f}", f"{meas[ph]:.6e}" if meas else ""])
        if solver is not None:
            w.writerow(["sync", str(solver.comm.sync_count), str(solver.comm.sync_volume),
                        str(solver.n_euler_steps)])


def report(solver, csv_path: Optional[str] = None, config: Optional[str] = None) -> str:
    """Report for a solver that has stepped with timers enabled (perf.py:147-153)."""
    text = format_table(solver.dim, card=solver.standard_card, solver=solver, config=config)
    if csv_path is not None:
        write_csv(csv_path, solver.dim, card=solver.standard_card, solver=solver)
    return text

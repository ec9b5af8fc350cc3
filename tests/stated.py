"""Loader for the stated-step-count reference digests (tests/golden/stated_*.json,
written by tests/golden/make_golden.py --stated from the UNMODIFIED reference)."""

import glob
import hashlib
import json
import os

import numpy as np

from paper_2007_00094_b200 import problems as P

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def stated_names():
    return sorted(os.path.basename(p)[len("stated_"):-5]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "stated_*.json")))


def load(name):
    with open(os.path.join(GOLDEN_DIR, f"stated_{name}.json")) as fh:
        return json.load(fh)


def input_digest(mat, U0, bc) -> str:
    """The same digest as make_golden.input_digest."""
    h = hashlib.sha256()
    arrs = [mat.indptr, mat.indices, mat.m, mat.c, mat.m_lumped, mat.inv_m, U0]
    if bc is not None:
        for a in (bc.inflow_nodes, bc.farfield, bc.slip_nodes, bc.slip_normals):
            if a is not None:
                arrs.append(a)
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def state_digest(U) -> str:
    return hashlib.sha256(np.ascontiguousarray(U).tobytes()).hexdigest()


def problem(rec):
    ps = getattr(P, rec["generator"])(*rec["args"])
    return ps


def run_and_compare(rec, solver, ps):
    """Drive `solver` (Solver-like) for the recorded steps; returns (taus, digests)."""
    solver.set_state(ps.U0)
    taus, dig = [], {}
    for k in range(1, rec["steps"] + 1):
        taus.append(solver.ssp_rk3_step())
        if str(k) in rec["state_sha256"]:
            dig[str(k)] = state_digest(solver.get_state())
    return taus, dig

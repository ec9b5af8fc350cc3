"""Loader for the reference-generated golden fixtures (tests/golden/*.npz)."""

import glob
import json
import os

import numpy as np

from paper_2007_00094_b200.problems import BoundaryConditions, PrecomputedMatrices

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith(("c1_full", "functions_")))


class Golden:
    def __init__(self, name):
        z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
        self.name = name
        self.z = z
        n, dim = int(z["n"]), int(z["dim"])
        m = z["m"]
        self.matrices = PrecomputedMatrices(
            n=n, dim=dim, indptr=z["indptr"], indices=z["indices"].astype(np.int64), m=m, c=z["c"],
            beta=np.zeros_like(m), m_lumped=z["m_lumped"], inv_m=z["inv_m"])
        self.U0 = z["U0"]
        bc = None
        if "bc_inflow" in z.files or "bc_slip" in z.files:
            bc = BoundaryConditions(
                inflow_nodes=z["bc_inflow"] if "bc_inflow" in z.files else None,
                farfield=z["bc_farfield"] if "bc_farfield" in z.files else None,
                slip_nodes=z["bc_slip"] if "bc_slip" in z.files else None,
                slip_normals=z["bc_normals"] if "bc_normals" in z.files else None)
        self.boundary = bc
        self.params = json.loads(str(z["params"]))
        self.taus = z["taus"]
        self.U_final = z["U_final"]

    def solver_kwargs(self):
        p = self.params
        return dict(c_cfl=p["c_cfl"], limiter_passes=p["passes"], newton_steps=p["newton"],
                    boundary=self.boundary)

    def run(self, solver):
        """Drive a Solver-like object through the recorded schedule."""
        solver.set_state(self.U0)
        taus = []
        tau = self.params.get("tau")
        for _ in range(self.params["steps"]):
            if self.params["mode"] == "euler":
                taus.append(solver.euler_step(tau))
            else:
                taus.append(solver.ssp_rk3_step(tau))
        return np.array(taus), solver.get_state()

    def internal(self, key):
        k = "int_" + key
        return self.z[k] if k in self.z.files else None

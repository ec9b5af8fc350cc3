"""BASELINE.json configurations at their FULL sizes.

Where the oracle finishes in seconds (C2: 1.23M nodes) the CUDA path is
compared with it bit-for-bit over a prefix of the run; everywhere else the
checks are size-independent properties of the scheme (arXiv 2007.00094 §3,
the reference's test_stepper.py:69-77 and test_acceptance.py criteria):

* conservation of mass, momentum and energy on the periodic box (C5, 320^3,
  32.8M nodes, one GPU), tolerance 1e-12 relative as test_stepper.py:69-77;
* the local invariant-domain bounds of every stage: rho_min_i <= rho_i <=
  rho_max_i and the specific-entropy minimum phi(U_i) >= phi_min_i, with the
  bounds the same stage computed, tolerance 1e-12 relative
  for rho and 1e-8 relative for phi (the limiter's Newton tolerance is 1e-10
  relative on rho*eps, limiter.py:39, 175);
* admissibility (rho > 0, eps > 0) at every node after every step (the
  library raises AdmissibilityError otherwise) over the full step counts.
"""

import os

import numpy as np
import pytest

import oracle as O
from paper_2007_00094_b200 import Solver
from paper_2007_00094_b200 import problems as P
from paper_2007_00094_b200.physics import AIR
from paper_2007_00094_b200.stepper import cm_permutation

pytestmark = pytest.mark.gpu


def _phi(U, dim):
    """phi = eps rho^-gamma with eps = E - |m|^2 / (2 rho) (physics.py:86-89, stepper.py:404)."""
    rho, E = U[:, 0], U[:, dim + 1]
    m2 = (U[:, 1:dim + 1] ** 2).sum(axis=1)
    eps = E - 0.5 * m2 / rho
    return eps * rho ** (-AIR.gamma), eps


def _stage_bounds_hold(s, dim, exclude_rows=()):
    """After one euler_step: the new state lies inside the bounds of that stage."""
    U = s.fetch("U")
    B = s.fetch("bounds")
    n = s.n_owned
    U, B = U[:n], B[:n]
    keep = np.ones(n, bool)
    keep[np.asarray(exclude_rows, dtype=np.int64)] = False
    rho = U[keep, 0]
    rmin, rmax, pmin = B[keep, 0], B[keep, 1], B[keep, 2]
    assert np.all(rho >= rmin - 1e-12 * np.abs(rmin)), float((rmin - rho).max())
    assert np.all(rho <= rmax + 1e-12 * np.abs(rmax)), float((rho - rmax).max())
    phi, eps = _phi(U[keep], dim)
    assert np.all(eps > 0.0) and np.all(rho > 0.0)
    assert np.all(phi >= pmin - 1e-8 * np.abs(pmin)), float(((pmin - phi) / np.abs(pmin)).max())


@pytest.fixture(scope="module")
def c2():
    return P.make_config("c2")


def test_c2_full_size_prefix_matches_oracle(c2):
    """Full C2 (1,234,310 nodes, 11.09M nnz): 4 SSP-RK3 steps bitwise equal to the oracle."""
    ps = c2
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    o = O.OracleSolver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary, threads=os.cpu_count() or 1)
    s.set_state(ps.U0)
    o.set_state(ps.U0)
    for k in range(4):
        t1, t2 = s.ssp_rk3_step(), o.ssp_rk3_step()
        assert t1 == t2, f"tau differs at step {k}"
    assert np.array_equal(s.get_state(), o.get_state())
    s.close()


def test_c2_full_run_invariants(c2):
    """Full C2, the benchmark's 200 steps: admissible throughout, and the local
    bounds of the last stage hold on every node but the inflow nodes (reset)."""
    ps = c2
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    s.set_state(ps.U0)
    for _ in range(199):
        s.ssp_rk3_step_async()
    s.sync()  # raises AdmissibilityError if any step produced an inadmissible state
    perm, _ = cm_permutation(ps.matrices)
    inflow_rows = perm[np.asarray(ps.boundary.inflow_nodes, dtype=np.int64)]
    s.euler_step()  # one more stage, its bounds are still in the work arrays
    _stage_bounds_hold(s, 2, exclude_rows=inflow_rows)
    U = s.get_state()
    assert np.all(np.isfinite(U))
    phi, eps = _phi(U, 2)
    assert np.all(U[:, 0] > 0) and np.all(eps > 0)
    s.close()


def test_c5_full_size_conservation_and_bounds():
    """Full C5 (320^3 periodic, 32.8M nodes, 885M nnz) on one GPU: mass, momentum
    and energy conserved to roundoff over 3 SSP-RK3 steps, stage bounds hold."""
    ps = P.make_config("c5")
    mat = ps.matrices
    s = Solver(mat, c_cfl=ps.c_cfl, boundary=ps.boundary)
    s.set_state(ps.U0)
    m = np.asarray(mat.m_lumped)
    tot0 = (m[:, None] * ps.U0).sum(axis=0)
    for _ in range(3):
        s.ssp_rk3_step()
    U = s.get_state()
    tot = (m[:, None] * U).sum(axis=0)
    scale = np.abs(m[:, None] * ps.U0).sum(axis=0)
    assert np.all(np.abs(tot - tot0) <= 1e-12 * scale), (tot - tot0) / scale
    s.euler_step()
    _stage_bounds_hold(s, 3)
    s.close()


def test_c2_full_run_fast_paths_are_exact(c2):
    """Full C2 over the benchmark's 200 steps: the default path (identical-state
    fast paths, frozen rows, d_ij memo, zero-P tags) and the general path give
    the same tau sequence and the same final state, bit for bit."""
    ps = c2
    runs = []
    for mode in (-1, 0):
        s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
        s.set_uniform_shortcuts(mode)
        s.set_state(ps.U0)
        taus = [s.ssp_rk3_step() for _ in range(200)]
        runs.append((taus, s.get_state()))
        s.close()
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("cfg,steps", [("c5m", 20), ("c3m", 20)])
def test_3d_limiter_fast_accept_is_exact(cfg, steps, monkeypatch):
    """3D: the limiter's fast accept (fp32 bound of the pow) on and off give the
    same run bit for bit (160^3 periodic box, 1.05M-node Sod box)."""
    ps = P.make_config(cfg)
    runs = []
    for fa in ("1", "0"):
        monkeypatch.setenv("EF_FAST_ACCEPT", fa)
        s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
        s.set_state(ps.U0)
        taus = [s.ssp_rk3_step() for _ in range(steps)]
        runs.append((taus, s.get_state()))
        s.close()
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])

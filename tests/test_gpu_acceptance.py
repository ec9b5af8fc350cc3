"""The reference's acceptance criteria (pkg/tests/test_acceptance.py) on the CUDA
Solver, with this package's problem generators (the reference's cylinder
channel mesh is replaced by the C2 disc channel at a small size):

* 01 invariant domain (:55-72): rho > 0 and eps > 0 after every RK step of
  the Mach-3 channel to t = 0.2 (hard-checked inside every stage as well);
* 02 entropy minimum principle (:76-97): with limiter_passes = 0 the specific
  entropy of every interior node stays above its stencil minimum (1e-12);
* 03 conservation (:101-114): periodic-smooth 64^2, 100 RK steps, relative
  drift of the lumped-mass totals <= 1e-11;
* 04 constant-state preservation (:118-127): bitwise after 10 RK steps;
* 10 accuracy ordering (:316-341): periodic-smooth at 32^2 / 64^2, the
  limited scheme is no less accurate than the low-order one and the low-order
  L1 error converges at rate >= 0.8."""

import numpy as np
import pytest

from paper_2007_00094_b200 import Solver
from paper_2007_00094_b200 import problems as P
from paper_2007_00094_b200.physics import AIR

pytestmark = pytest.mark.gpu


def _eps(U):
    return U[:, -1] - 0.5 * (U[:, 1:-1] ** 2).sum(axis=1) / U[:, 0]


def _entropy(U):  # physics.specific_entropy (physics.py:106-114): log(e) / gm1 - log(rho)
    return np.log(_eps(U) / U[:, 0]) / AIR.gm1 - np.log(U[:, 0])


def test_criterion_01_invariant_domain():
    ps = P.mach3_disc(60, seed=1)
    s = Solver(ps.matrices, c_cfl=0.9, limiter_passes=2, boundary=ps.boundary)
    s.set_state(ps.U0)
    worst = [np.inf]

    def check(step, t):
        U = s.get_state()
        worst[0] = min(worst[0], U[:, 0].min(), _eps(U).min())

    steps = s.advance(0.2, on_step=check)
    assert steps > 10 and worst[0] > 0.0


def test_criterion_02_entropy_minimum_principle():
    ps = P.mach3_disc(40, seed=2)
    mat = ps.matrices
    s = Solver(mat, c_cfl=0.9, limiter_passes=0, boundary=ps.boundary)
    s.set_state(ps.U0)
    interior = np.ones(mat.n, dtype=bool)
    interior[ps.boundary.inflow_nodes] = False
    interior[ps.boundary.slip_nodes] = False
    t, worst = 0.0, np.inf
    while t < 0.1 - 1e-14:
        ent_old = _entropy(s.get_state())
        stencil_min = np.minimum.reduceat(ent_old[mat.indices], mat.indptr[:-1])
        t += s.euler_step(tau_max=0.1 - t)
        slack = (_entropy(s.get_state()) - stencil_min)[interior]
        worst = min(worst, slack.min())
    assert worst >= -1e-12


def test_criterion_03_conservation():
    ps = P.periodic_smooth(n=64)
    mat = ps.matrices
    s = Solver(mat)
    s.set_state(ps.U0)
    before = (mat.m_lumped[:, None] * ps.U0).sum(axis=0)
    for _ in range(100):
        s.ssp_rk3_step()
    after = (mat.m_lumped[:, None] * s.get_state()).sum(axis=0)
    scale = np.maximum(np.abs(before), np.abs(before).max())
    assert (np.abs(after - before) / scale).max() <= 1e-11


def test_criterion_04_constant_state_preservation():
    mat = P.assemble_q1(P.rectangle_mesh(8, 8, periodic=(True, True)))
    U = np.tile([1.4, 4.2, -1.1, 8.8], (mat.n, 1))
    s = Solver(mat)
    s.set_state(U)
    for _ in range(10):
        s.ssp_rk3_step()
    assert np.array_equal(s.get_state(), U)


def test_criterion_10_accuracy_ordering():
    t_final = 0.05
    errors = {}
    for n in (32, 64):
        ps = P.periodic_smooth(n=n)
        mat = ps.matrices
        pts = np.zeros((mat.n, 2))
        pts[ps.mesh.reduced_index] = ps.mesh.points
        U_ref = ps.exact(pts, t_final)
        for passes in (0, 2):
            s = Solver(mat, limiter_passes=passes)
            s.set_state(ps.U0)
            s.advance(t_final)
            errors[(n, passes)] = (mat.m_lumped * np.abs(s.get_state()[:, 0] - U_ref[:, 0])).sum()
    assert errors[(32, 2)] <= errors[(32, 0)]
    assert errors[(64, 2)] <= errors[(64, 0)]
    assert np.log2(errors[(32, 0)] / errors[(64, 0)]) >= 0.8

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
* 05 Riemann bound (:131-159): the device lambda_max >= the exact wave speed
  (own exact Riemann solver: pressure function, bisection), identical pairs;
* 06 limiter optimality (:163-200): device factors feasible and within 1e-6
  of the largest feasible factor (scan + bisection) where the bound is active;
* 10 accuracy ordering (:316-341): periodic-smooth at 32^2 / 64^2, the
  limited scheme is no less accurate than the low-order one and the low-order
  L1 error converges at rate >= 0.8.
Criteria 07 (quadratic Newton step) and 08 (storage equivalence) test
reference-internal helpers; the device versions are covered bitwise by the
function-level goldens (test_gpu_functions.py) and the parity tests; 09 is
test_gpu_multirank.py, 12 the RK3 parity of test_gpu_parity.py."""

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


# ----- 05 / 06: the device Riemann bound and limiter against exact solutions ------

def _random_states(rng, count, dim=2):  # ranges of test_acceptance.py:28-35
    U = np.zeros((count, dim + 2))
    U[:, 0] = 0.1 + 1.9 * rng.random(count)
    vel = rng.normal(0.0, 1.5, (count, dim))
    U[:, 1:-1] = U[:, 0:1] * vel
    p = 0.05 + 2.0 * rng.random(count)
    U[:, -1] = p / AIR.gm1 + 0.5 * U[:, 0] * (vel ** 2).sum(axis=1)
    return U, vel, p


def _exact_lambda(rl, ul, pl, rr, ur, pr, g=AIR.gamma):
    """Exact extreme wave speeds of the 1D Riemann problem: p* from the pressure
    function f_L(p) + f_R(p) + (u_R - u_L) = 0 (shock / rarefaction branches,
    increasing in p) by bisection in log p; vacuum -> the acoustic speeds."""
    cl, cr = np.sqrt(g * pl / rl), np.sqrt(g * pr / rr)

    def f(p, rho, pk, ck):
        shock = (p - pk) * np.sqrt((2.0 / ((g + 1.0) * rho)) / (p + (g - 1.0) / (g + 1.0) * pk))
        rare = (2.0 * ck / (g - 1.0)) * ((p / pk) ** ((g - 1.0) / (2.0 * g)) - 1.0)
        return np.where(p > pk, shock, rare)

    def phi(p):
        return f(p, rl, pl, cl) + f(p, rr, pr, cr) + (ur - ul)

    lo = np.full_like(pl, 1e-300)
    hi = np.maximum(pl, pr)
    for _ in range(200):  # bracket from above
        grow = phi(hi) < 0.0
        if not grow.any():
            break
        hi = np.where(grow, hi * 4.0, hi)
    vacuum = phi(lo) > 0.0
    for _ in range(1100):
        mid = np.sqrt(lo * hi)
        neg = phi(mid) < 0.0
        lo, hi = np.where(neg, mid, lo), np.where(neg, hi, mid)
    ps = 0.5 * (lo + hi)
    gp = (g + 1.0) / (2.0 * g)
    lam1 = ul - cl * np.sqrt(1.0 + gp * np.maximum((ps - pl) / pl, 0.0))
    lam3 = ur + cr * np.sqrt(1.0 + gp * np.maximum((ps - pr) / pr, 0.0))
    lam = np.maximum(np.maximum(-lam1, 0.0), np.maximum(lam3, 0.0))
    acoustic = np.maximum(np.maximum(-(ul - cl), 0.0), np.maximum(ur + cr, 0.0))
    return np.where(vacuum, acoustic, lam)


def test_criterion_05_riemann_bound():
    """test_acceptance.py:131-159: the device lambda_max bound (d_ij of a unit c
    with a zero c_ji, i.e. lambda(n; U_L, U_R)) is >= the exact wave speed, and
    the identical-state pair gives |u.n| + c."""
    from paper_2007_00094_b200.stepper import eval_dij

    rng = np.random.default_rng(2024)
    n_pairs = 10_000
    UL, velL, pL = _random_states(rng, n_pairs)
    UR, velR, pR = _random_states(rng, n_pairs)
    n = rng.normal(size=(n_pairs, 2))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    bound, bad = eval_dij(UL, UR, n, np.zeros_like(n))
    assert not bad.any()
    exact = _exact_lambda(UL[:, 0], (velL * n).sum(1), pL, UR[:, 0], (velR * n).sum(1), pR)
    assert (bound - exact).min() >= -1e-12
    same, _ = eval_dij(UL, UL, n, np.zeros_like(n))
    expect = np.abs((velL * n).sum(axis=1)) + np.sqrt(AIR.gamma * pL / UL[:, 0])
    assert np.abs(same - expect).max() <= 1e-10


def _limiter_cases(rng, count, dim=2):  # test_acceptance.py:38-52, vectorized
    st = np.zeros((count, 6, dim + 2))
    st[..., 0] = 0.3 + 1.5 * rng.random((count, 6))
    st[..., 1:-1] = rng.normal(0.0, 0.5, (count, 6, dim)) * st[..., 0:1]
    p = 0.2 + rng.random((count, 6))
    st[..., -1] = p / AIR.gm1 + 0.5 * (st[..., 1:-1] ** 2).sum(-1) / st[..., 0]
    phi = (st[..., -1] - 0.5 * (st[..., 1:-1] ** 2).sum(-1) / st[..., 0]) * st[..., 0] ** (-AIR.gamma)
    P = rng.normal(0.0, 0.4, (count, dim + 2))
    bounds = np.column_stack([st[..., 0].min(1), st[..., 0].max(1), phi.min(1)])
    return st[:, 0], P, bounds


def test_criterion_06_limiter_optimality():
    """test_acceptance.py:163-200: every factor of the device limiter (4 Newton
    steps) is feasible, never above the largest feasible factor found by a scan
    plus bisection, and within 1e-6 of it where the bound is active."""
    from paper_2007_00094_b200.stepper import eval_limiter

    rng = np.random.default_rng(4096)
    U, P, bnd = _limiter_cases(rng, 10_000)
    t4 = eval_limiter(U, P, bnd, newton_steps=4)
    g = AIR.gamma
    re0 = U[:, 0] * U[:, -1] - 0.5 * (U[:, 1:-1] ** 2).sum(1)
    tol = 1e-10 * np.abs(re0)
    rtol = 1e-12 * np.maximum(np.maximum(np.abs(bnd[:, 0]), np.abs(bnd[:, 1])), 1.0)

    def psi(t):  # (rho < 0 only at infeasible scan points: NaN there counts as infeasible)
        V = U + t[:, None] * P
        with np.errstate(invalid="ignore"):
            return V, V[:, 0] * V[:, -1] - 0.5 * (V[:, 1:-1] ** 2).sum(1) - bnd[:, 2] * V[:, 0] ** (g + 1.0)

    def feasible(t):
        V, ps = psi(t)
        return (V[:, 0] >= bnd[:, 0] - rtol) & (V[:, 0] <= bnd[:, 1] + rtol) & (ps >= -tol)

    V, ps = psi(t4)
    assert ((t4 >= 0) & (t4 <= 1)).all()
    assert ((V[:, 0] >= bnd[:, 0] - 1e-11) & (V[:, 0] <= bnd[:, 1] + 1e-11) & (ps >= -tol)).all()
    # largest feasible factor: first infeasible point of a 512-point scan, then bisection
    ts = np.linspace(0.0, 1.0, 513)
    first_bad = np.full(len(U), 513)
    for k in range(512, 0, -1):
        first_bad = np.where(~feasible(np.full(len(U), ts[k])), k, first_bad)
    t_ref = np.ones(len(U))
    has = first_bad < 513
    lo = np.where(has, ts[np.maximum(first_bad - 1, 0)], 1.0)
    hi = np.where(has, ts[np.minimum(first_bad, 512)], 1.0)
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        ok = feasible(mid)
        lo, hi = np.where(ok, mid, lo), np.where(ok, hi, mid)
    t_ref = np.where(has, lo, 1.0)
    t_ref = np.where(feasible(np.zeros(len(U))), t_ref, 0.0)
    assert (t4 <= t_ref + 1e-9).all()
    _, psi0 = psi(np.zeros(len(U)))
    active = (psi0 > tol) & (t_ref < 1.0 - 1e-9)
    assert active.sum() > 1000
    assert np.abs(t4 - t_ref)[active].max() <= 1e-6

"""CUDA path vs the pinned oracle / the reference goldens — bit-for-bit.

Tolerance: zero.  Every comparison is np.array_equal (and tau ==), because the
kernels reproduce the reference's fp64 operation sequence exactly once the
shared pow is installed on both sides."""

import numpy as np
import pytest

import oracle as O
from goldens import Golden, names
from paper_2007_00094_b200 import Solver
from paper_2007_00094_b200 import problems as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", names())
def test_gpu_matches_reference_golden(name):
    g = Golden(name)
    s = Solver(g.matrices, **g.solver_kwargs())
    taus, U = g.run(s)
    assert np.array_equal(taus, g.taus)
    assert np.array_equal(U, g.U_final)


def _internals_cm(s, keys=("d", "alpha", "R", "bounds")):
    gids = s.local_gids()
    out = {}
    for key in keys:
        a = s.fetch(key)
        b = np.empty_like(a)
        b[gids] = a
        out[key] = b
    return out


@pytest.mark.parametrize("name", [n for n in names() if n.endswith("euler") or "_euler_" in n])
def test_gpu_first_stage_internals(name):
    g = Golden(name)
    s = Solver(g.matrices, **g.solver_kwargs())
    s.set_state(g.U0)
    s.euler_step(g.params.get("tau"))
    got = _internals_cm(s)
    ref_d = g.internal("d")
    assert np.array_equal(got["d"], ref_d)
    assert np.array_equal(got["alpha"], g.internal("alpha"))
    assert np.array_equal(got["R"], g.internal("R"))
    assert np.array_equal(got["bounds"], g.internal("bounds"))


def _transpose_slots(mat):
    """(row, slot) -> (row, slot) of the transposed entry, rows and slots in the
    global CM order the reference uses (stepper.py:195-236)."""
    cm_perm, _ = O.cm_permutation(mat)
    n = mat.n
    rows = [[] for _ in range(n)]
    for o in range(n):
        rows[cm_perm[o]] = sorted(int(cm_perm[c]) for c in mat.indices[mat.indptr[o]:mat.indptr[o + 1]])
    pos = [{c: t for t, c in enumerate(r)} for r in rows]
    return rows, pos


@pytest.mark.parametrize("name", [n for n in names() if n.endswith("euler") or "_euler_" in n])
def test_gpu_first_stage_P_and_limiter_factors(name):
    """The reference's rk.P after the first stage (the correction fluxes of its last
    limiter pass) bit for bit, and -- on the edges the last pass limits (previous
    factor below 1) -- min(l_ij, l_ji) of the reference's last-pass factors rk.l.
    General path (identical-state shortcuts off: their zero-P tags do not keep
    the sign of a zero P)."""
    g = Golden(name)
    s = Solver(g.matrices, **g.solver_kwargs())
    s.set_uniform_shortcuts(0)
    s.set_state(g.U0)
    s.euler_step(g.params.get("tau"))
    got = _internals_cm(s, ("P", "l", "l_prev"))
    if g.params["passes"] == 0:
        return
    refP = g.internal("P")
    bad = np.argwhere(got["P"].view(np.int64) != refP.view(np.int64))
    assert len(bad) == 0, (len(bad), [(tuple(b), got["P"][tuple(b)], refP[tuple(b)],
                                       got["l_prev"][tuple(b[:2])]) for b in bad[:6]])
    if g.params["passes"] != 2:
        return
    rows, pos = _transpose_slots(g.matrices)
    ref_l = g.internal("l")
    for i, cols in enumerate(rows):
        for sl, j in enumerate(cols):
            if j <= i or not (0.0 <= got["l_prev"][i, sl] < 1.0):
                continue  # the last pass limits only edges whose previous factor was below 1
            t = pos[j][i]
            want = min(ref_l[i, sl], ref_l[j, t])
            assert got["l"][i, sl] == want and got["l"][j, t] == want, (i, sl)


def _compare(ps_matrices, U0, bc, steps, c_cfl=0.9, passes=2, newton=2, threads=8):
    s = Solver(ps_matrices, c_cfl=c_cfl, limiter_passes=passes, newton_steps=newton, boundary=bc)
    o = O.OracleSolver(ps_matrices, c_cfl=c_cfl, limiter_passes=passes, newton_steps=newton,
                       boundary=bc, threads=threads)
    s.set_state(U0)
    o.set_state(U0)
    for k in range(steps):
        t1 = s.ssp_rk3_step()
        t2 = o.ssp_rk3_step()
        assert t1 == t2, f"tau differs at step {k}"
    a, b = s.get_state(), o.get_state()
    assert np.array_equal(a, b), f"max |dU| = {np.abs(a - b).max():.3e}"
    return a


def test_gpu_c1_full_size_100_steps():
    ps = P.isentropic_vortex(128)
    _compare(ps.matrices, ps.U0, ps.boundary, 100, c_cfl=0.5)


@pytest.mark.parametrize("ny", [20, 60])
def test_gpu_c2_disc(ny):
    ps = P.mach3_disc(ny, seed=ny)
    _compare(ps.matrices, ps.U0, ps.boundary, 10)


def test_gpu_c3_sod_box():
    ps = P.sod_box(31, 7, 7, seed=9)
    _compare(ps.matrices, ps.U0, ps.boundary, 8)


def test_gpu_c4_cylinder():
    ps = P.mach3_cylinder(20, 6, seed=8)
    _compare(ps.matrices, ps.U0, ps.boundary, 3)


def test_gpu_c5_periodic_box():
    ps = P.periodic_fourier_box(12, seed=4)
    _compare(ps.matrices, ps.U0, None, 5)


@pytest.mark.parametrize("passes,newton", [(0, 2), (1, 2), (3, 1), (2, 4)])
def test_gpu_limiter_variants(passes, newton):
    ps = P.mach3_disc(20, seed=3)
    _compare(ps.matrices, ps.U0, ps.boundary, 4, passes=passes, newton=newton)


def test_gpu_random_fields_3d():
    mat = P.assemble_q1(P.box_mesh(6, 5, 4, periodic=(True, True, True)))
    U = P.random_state(np.random.default_rng(2024), mat.n, dim=3)
    _compare(mat, U, None, 3)


def _blocky_state(rng, mat, dim, nblocks, negzero=True):
    """Piecewise-constant random states: many edges join identical states (the
    identical-state and zero-correction shortcuts), the rest are block interfaces;
    some blocks at rest with -0 momentum components."""
    U = np.empty((mat.n, dim + 2))
    lab = rng.integers(0, nblocks, mat.n)
    # spatially coherent labels: smooth the random labels along the node order
    lab = np.repeat(lab[:: max(1, mat.n // (4 * nblocks))], max(1, mat.n // (4 * nblocks)))[: mat.n]
    lab = np.concatenate([lab, np.zeros(mat.n - len(lab), dtype=lab.dtype)])
    states = P.random_state(rng, nblocks, dim=dim)
    if negzero:
        states[0, 1:-1] = -0.0
        states[1, 1] = -0.0
    U[:] = states[lab]
    return U


@pytest.mark.parametrize("dim", [2, 3])
def test_gpu_blocky_states_bitwise(dim):
    rng = np.random.default_rng(77 + dim)
    mesh = P.rectangle_mesh(40, 30, periodic=(True, True)) if dim == 2 else \
        P.box_mesh(12, 10, 8, periodic=(True, True, True))
    mat = P.assemble_q1(mesh)
    U = _blocky_state(rng, mat, dim, 6)
    for passes in (2, 3):
        _compare(mat, U, None, 4, passes=passes)


@pytest.mark.parametrize("mode", ["0", "1"])
def test_gpu_identical_state_shortcuts_forced(mode, monkeypatch):
    """The identical-state shortcuts forced off and on give the oracle's bits
    (the default chooses per step from the count of identical-state edges)."""
    monkeypatch.setenv("EF_UNIFORM", mode)
    ps = P.mach3_disc(20, seed=5)
    _compare(ps.matrices, ps.U0, ps.boundary, 6)
    rng = np.random.default_rng(5)
    mat = P.assemble_q1(P.box_mesh(10, 8, 6, periodic=(True, True, True)))
    _compare(mat, _blocky_state(rng, mat, 3, 5), None, 3)


def test_gpu_frozen_rows_with_ulp_energy_perturbation():
    """A gas at rest with uniform density and energy perturbed by a few ulps at
    a few nodes: rows next to the perturbed ones have uniform stencils, get
    limited updates of ~1 ulp that the RK combination can round away, and must
    not be frozen with a stale U^L.  Shortcuts forced on == off ==
    oracle, bit for bit."""
    mat = P.assemble_q1(P.rectangle_mesh(24, 24, periodic=(True, True)))
    U = np.tile([1.0, 0.0, 0.0, 2.5], (mat.n, 1))
    rng = np.random.default_rng(11)
    for k in rng.choice(mat.n, 12, replace=False):
        for _ in range(int(rng.integers(1, 4))):
            U[k, 3] = np.nextafter(U[k, 3], np.inf if rng.random() < 0.5 else -np.inf)
    res = []
    for mode in (1, 0):
        s = Solver(mat)
        s.set_uniform_shortcuts(mode)
        s.set_state(U)
        taus = [s.ssp_rk3_step(tau=1e-3) for _ in range(12)]
        res.append((taus, s.get_state()))
    o = O.OracleSolver(mat)
    o.set_state(U)
    taus_o = [o.ssp_rk3_step(1e-3) for _ in range(12)]
    assert res[0][0] == res[1][0] == taus_o
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][1], o.get_state())

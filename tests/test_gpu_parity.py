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


def _internals_cm(s):
    gids = s.local_gids()
    out = {}
    for key in ("d", "alpha", "R", "bounds"):
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

"""The multi-rank path (contiguous CM ranges, ghost rows with truncated
stencils, halo exchanges of alpha / R / l / U, tau min-reduction) run as a
same-device group: results must be bitwise identical to one rank, as the
reference asserts for its simulated ranks (test_acceptance.py:293-311,
test_stepper.py:106-128)."""

import numpy as np
import pytest

import oracle as O
from goldens import Golden
from paper_2007_00094_b200 import Solver
from paper_2007_00094_b200 import problems as P

pytestmark = pytest.mark.gpu


def _run(mat, U0, bc, ranks, steps, mode="rk3", **kw):
    s = Solver(mat, boundary=bc, ranks=ranks, **kw)
    s.set_state(U0)
    taus = [s.ssp_rk3_step() if mode == "rk3" else s.euler_step() for _ in range(steps)]
    return taus, s.get_state(), s


CASES = {
    "c1": lambda: P.isentropic_vortex(24),
    "c2": lambda: P.mach3_disc(20, seed=7),
    "c3": lambda: P.sod_box(15, 4, 4, seed=3),
    "c5": lambda: P.periodic_fourier_box(8, seed=2),
    "c4": lambda: P.mach3_cylinder(10, 3, seed=6),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("ranks", [2, 3, 5])
@pytest.mark.parametrize("overlap", [True, False])
def test_ranks_are_bitwise_identical(case, ranks, overlap):
    ps = CASES[case]()
    t1, U1, _ = _run(ps.matrices, ps.U0, ps.boundary, 1, 4, c_cfl=ps.c_cfl)
    tR, UR, s = _run(ps.matrices, ps.U0, ps.boundary, ranks, 4, c_cfl=ps.c_cfl, overlap=overlap)
    assert t1 == tR
    assert np.array_equal(U1, UR)
    assert s.comm.sync_count > 0 and s.comm.sync_volume > 0


@pytest.mark.parametrize("overlap", [True, False])
def test_overlap_with_interior_rows(overlap):
    """Ranks large enough that exported rows are a small prefix/suffix of the
    range: the interior launches and the comm-stream halos both run."""
    ps = P.mach3_disc(80, seed=5)
    t1, U1, _ = _run(ps.matrices, ps.U0, ps.boundary, 1, 5)
    t4, U4, s = _run(ps.matrices, ps.U0, ps.boundary, 4, 5, overlap=overlap)
    assert t1 == t4 and np.array_equal(U1, U4)
    # per stage: alpha, (R, U^L, bounds), U^L after pass 0, U -- one message each
    assert s.comm.sync_count == 4 * 3 * 5


@pytest.mark.parametrize("passes", [0, 1, 3])
def test_ranks_with_limiter_variants(passes):
    ps = P.mach3_disc(20, seed=9)
    t1, U1, _ = _run(ps.matrices, ps.U0, ps.boundary, 1, 3, limiter_passes=passes)
    t4, U4, _ = _run(ps.matrices, ps.U0, ps.boundary, 4, 3, limiter_passes=passes)
    assert t1 == t4 and np.array_equal(U1, U4)


def test_ranks_match_reference_golden():
    g = Golden("mach3_channel_r2")
    s = Solver(g.matrices, ranks=3, **g.solver_kwargs())
    taus, U = g.run(s)
    assert np.array_equal(taus, g.taus) and np.array_equal(U, g.U_final)


def test_ranks_euler_and_roundtrip():
    ps = P.sod_box(11, 3, 3, seed=4)
    s = Solver(ps.matrices, boundary=ps.boundary, ranks=4)
    s.set_state(ps.U0)
    assert np.array_equal(s.get_state(), ps.U0)
    o = O.OracleSolver(ps.matrices, boundary=ps.boundary)
    o.set_state(ps.U0)
    for _ in range(3):
        assert s.euler_step() == o.euler_step()
    assert np.array_equal(s.get_state(), o.get_state())


@pytest.mark.parametrize("mode", ["0", "1"])
@pytest.mark.parametrize("case", ["c2", "c3"])
def test_ranks_identical_state_shortcuts_forced(mode, case, monkeypatch):
    """Shortcuts forced off / on: ghost rows never take them (their stencils are
    truncated), the halo data are the same, so every rank count agrees."""
    monkeypatch.setenv("EF_UNIFORM", mode)
    ps = CASES[case]()
    t1, U1, _ = _run(ps.matrices, ps.U0, ps.boundary, 1, 4, c_cfl=ps.c_cfl)
    t3, U3, _ = _run(ps.matrices, ps.U0, ps.boundary, 3, 4, c_cfl=ps.c_cfl)
    assert t1 == t3 and np.array_equal(U1, U3)


def test_eight_ranks_c5_64_with_overlap():
    """The 8-GPU shape on one device: C5 at 64^3 split into 8 CM ranges,
    overlap on, bitwise equal to one rank."""
    ps = P.periodic_fourier_box(64)
    t1, U1, _ = _run(ps.matrices, ps.U0, None, 1, 3)
    t8, U8, s = _run(ps.matrices, ps.U0, None, 8, 3, overlap=True)
    assert t1 == t8 and np.array_equal(U1, U8)


# ---- per-rank setup (ShardedSolver / ef_create_local) -------------------------
from paper_2007_00094_b200.distributed import ShardedSolver  # noqa: E402


def _box_global(n, steps, **kw):
    """One rank, the global periodic box matrices in their lexicographic order
    (identity permutation: the order the per-rank generator uses)."""
    ps = P.periodic_fourier_box(n)
    s = Solver(ps.matrices, cm_perm=np.arange(ps.matrices.n), **kw)
    s.set_state(ps.U0)
    taus = [s.ssp_rk3_step() for _ in range(steps)]
    return ps, taus, s.get_state()


@pytest.mark.parametrize("ranks", [2, 3, 8])
@pytest.mark.parametrize("overlap", [True, False])
def test_sharded_ranks_equal_one_rank(ranks, overlap):
    """Every rank built from its own rows (no global matrix): bitwise equal to
    one rank built from the global matrices in the same node order."""
    n, steps = 16, 4
    ps, t1, U1 = _box_global(n, steps)
    parts = [P.periodic_box_local(n, r, ranks) for r in range(ranks)]
    s = ShardedSolver(parts, overlap=overlap)
    s.set_state(ps.U0)
    tR = [s.ssp_rk3_step() for _ in range(steps)]
    assert t1 == tR
    assert np.array_equal(U1, s.get_state())
    assert s.comm.sync_count > 0


def test_sharded_single_rank_and_oracle_in_box_order():
    """R = 1 per-rank setup == global setup == the oracle with the same order."""
    n, steps = 12, 3
    ps, t1, U1 = _box_global(n, steps)
    s = ShardedSolver([P.periodic_box_local(n, 0, 1)])
    s.set_state(ps.U0)
    assert [s.ssp_rk3_step() for _ in range(steps)] == t1
    assert np.array_equal(s.get_state(), U1)
    o = O.OracleSolver(ps.matrices, cm_perm=np.arange(ps.matrices.n))
    o.set_state(ps.U0)
    assert [o.ssp_rk3_step() for _ in range(steps)] == t1
    assert np.array_equal(o.get_state(), U1)


def test_sharded_rejects_inadmissible_state_on_every_rank():
    n, R = 8, 3
    ps = P.periodic_fourier_box(n)
    s = ShardedSolver([P.periodic_box_local(n, r, R) for r in range(R)])
    s.set_state(ps.U0)
    bad = ps.U0.copy()
    bad[n ** 3 - 5, 0] = -1.0  # owned by the last rank, a ghost of rank 0 (periodic wrap)
    with pytest.raises(ValueError):
        s.set_state(bad)
    assert np.array_equal(s.get_state(), ps.U0)


@pytest.mark.parametrize("overlap", [True, False])
def test_group_graph_replay_is_bitwise_identical(overlap):
    """Multi-rank steps (halo copies on the comm stream, tau min over the
    ranks) captured into CUDA graphs and replayed equal direct launches; the
    halo statistics are re-added per replay."""
    ps = P.mach3_disc(30, seed=4)
    runs = []
    for graphs in (True, False):
        s = Solver(ps.matrices, boundary=ps.boundary, ranks=3, overlap=overlap)
        s.enable_graphs(graphs)
        s.set_state(ps.U0)
        taus = [s.ssp_rk3_step() for _ in range(4)] + [s.euler_step(tau=1e-4)]
        runs.append((taus, s.get_state(), s.comm.sync_count, s.comm.sync_volume, s.n_euler_steps))
    (ta, Ua, ca, va, na), (tb, Ub, cb, vb, nb) = runs
    assert ta == tb and np.array_equal(Ua, Ub)
    assert (ca, va, na) == (cb, vb, nb)


@pytest.mark.parametrize("ranks", [2, 4])
def test_sharded_c4_equals_one_rank(ranks):
    """C4 built per rank (z-slabs of the extruded O-grid, slip walls, inflow,
    outflow) steps bitwise like one rank built from the global matrices in the
    same (layer-major) node order."""
    ny, nz, steps = 10, 6, 3
    g = P.mach3_cylinder(ny, nz, shuffle=False)
    s1 = Solver(g.matrices, boundary=g.boundary, cm_perm=np.arange(g.matrices.n))
    s1.set_state(g.U0)
    t1 = [s1.ssp_rk3_step() for _ in range(steps)]
    parts = [P.mach3_cylinder_local(ny, nz, r, ranks) for r in range(ranks)]
    s = ShardedSolver([p.local for p in parts], boundary=g.boundary)
    s.set_state(g.U0)
    assert [s.ssp_rk3_step() for _ in range(steps)] == t1
    assert np.array_equal(s.get_state(), s1.get_state())

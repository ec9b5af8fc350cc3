"""The reference's Solver tests (pkg/tests/test_stepper.py) against the CUDA Solver."""

import numpy as np
import pytest

import oracle as O
from paper_2007_00094_b200 import AdmissibilityError, Solver, compute_tau, shared_pow
from paper_2007_00094_b200 import _lib
from paper_2007_00094_b200 import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small_periodic():
    mat = P.assemble_q1(P.rectangle_mesh(4, 4, periodic=(True, True)))
    return mat, P.random_state(np.random.default_rng(7), mat.n)


def test_constant_state_is_exactly_preserved(small_periodic):  # test_stepper.py:59-66
    mat, _ = small_periodic
    U = np.tile([1.4, 4.2, 0.0, 8.8], (mat.n, 1))
    s = Solver(mat)
    s.set_state(U)
    tau = s.euler_step()
    assert np.isfinite(tau) and tau > 0.0
    assert np.array_equal(s.get_state(), U)


def test_conservation_short_run(small_periodic):  # test_stepper.py:69-77
    mat, U = small_periodic
    s = Solver(mat)
    s.set_state(U)
    before = (mat.m_lumped[:, None] * U).sum(axis=0)
    for _ in range(5):
        s.ssp_rk3_step()
    after = (mat.m_lumped[:, None] * s.get_state()).sum(axis=0)
    assert np.abs(after - before).max() < 1e-12 * np.abs(before).max()


def test_state_roundtrip(small_periodic):  # test_stepper.py:80-84
    mat, U = small_periodic
    s = Solver(mat, ranks=3)
    s.set_state(U)
    assert np.array_equal(s.get_state(), U)


def test_rejects_inadmissible_initial_state(small_periodic):  # test_stepper.py:87-93
    mat, U = small_periodic
    bad = U.copy()
    bad[3, 0] = -1.0
    s = Solver(mat)
    s.set_state(U)
    with pytest.raises(AdmissibilityError):
        s.set_state(bad)
    assert np.array_equal(s.get_state(), U)  # state untouched


def test_invalid_parameters(small_periodic):  # test_stepper.py:96-103
    mat, _ = small_periodic
    for kw in (dict(c_cfl=0.0), dict(c_cfl=1.5), dict(limiter_passes=-1)):
        with pytest.raises(ValueError):
            Solver(mat, **kw)


def test_worker_lane_rank_arguments_do_not_change_results(small_periodic):  # :106-128
    mat, U = small_periodic
    outs = []
    for kw in (dict(), dict(ranks=3), dict(workers=2, chunk_size=3), dict(lanes=1), dict(overlap=False)):
        s = Solver(mat, **kw)
        s.set_state(U)
        s.ssp_rk3_step()
        outs.append(s.get_state())
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


def test_ssp_rk3_composition(small_periodic):  # test_stepper.py:131-147
    mat, U = small_periodic
    s = Solver(mat)
    s.set_state(U)
    tau = s.ssp_rk3_step()
    s2 = Solver(mat)
    s2.set_state(U)
    assert s2.euler_step() == tau
    U1 = s2.get_state()
    s2.set_state(U1)
    s2.euler_step(tau)
    U2 = 0.75 * U + 0.25 * s2.get_state()
    s2.set_state(U2)
    s2.euler_step(tau)
    U3 = U / 3.0 + (2.0 / 3.0) * s2.get_state()
    assert np.allclose(s.get_state(), U3, rtol=1e-14, atol=1e-14)


def test_advance_hits_final_time(small_periodic):  # test_stepper.py:150-156
    mat, U = small_periodic
    s = Solver(mat)
    s.set_state(U)
    taus = []
    s.advance(0.02, on_step=lambda k, t: taus.append(s.tau_last))
    assert abs(sum(taus) - 0.02) < 1e-13


def test_slip_wall_and_inflow():  # test_stepper.py:159-173
    ps = P.mach3_disc(20, seed=1)
    s = Solver(ps.matrices, boundary=ps.boundary)
    s.set_state(ps.U0)
    s.euler_step()
    U = s.get_state()
    bc = ps.boundary
    mom = U[bc.slip_nodes][:, 1:3]
    assert np.abs((mom * bc.slip_normals).sum(axis=1)).max() < 1e-13
    assert np.array_equal(U[bc.inflow_nodes], np.tile(bc.farfield, (len(bc.inflow_nodes), 1)))


def test_alpha_zero_on_constant_state(small_periodic):  # test_stepper.py:176-182
    mat, _ = small_periodic
    U = np.tile([1.0, 0.3, -0.2, 3.0], (mat.n, 1))
    s = Solver(mat)
    s.set_state(U)
    s.euler_step(tau=1e-3)
    assert np.abs(s.fetch("alpha")).max() == 0.0


def test_tau_equals_compute_tau(small_periodic):  # test_stepper.py:43-51
    mat, U = small_periodic
    s = Solver(mat, c_cfl=0.5)
    s.set_state(U)
    tau = s.euler_step()
    d = s.fetch("d")
    L = s.pad_width
    gids = s.local_gids()
    card = np.diff(mat.indptr)
    # diagonal slot of each local row
    o = O.OracleSolver(mat, c_cfl=0.5)
    o.set_state(U)
    o.euler_step()
    dd = o.fetch("d")
    diag = np.array([np.flatnonzero(o.fetch("d")[i] < 0)[0] for i in range(mat.n)])
    d_diag = dd[np.arange(mat.n), diag]
    m_cm = mat.m_lumped[o.cm_inv]
    assert tau == compute_tau(d_diag, m_cm, 0.5)


def test_unbounded_tau_raises(small_periodic):
    import dataclasses
    mat, U = small_periodic
    flat = dataclasses.replace(mat, c=np.zeros_like(mat.c))
    s = Solver(flat)
    s.set_state(U)
    with pytest.raises(ValueError):
        s.euler_step()
    assert np.array_equal(s.get_state(), U)


def test_timers_and_counters(small_periodic):  # test_stepper.py:185-194
    mat, U = small_periodic
    s = Solver(mat)
    s.enable_timers(True)
    s.set_state(U)
    s.ssp_rk3_step()
    assert s.n_euler_steps == 3
    t = s.timers
    assert all(v >= 0.0 for v in t.values()) and t["step1"] > 0.0 and t["step3"] > 0.0


def test_device_pow_equals_host_pow():
    rng = np.random.default_rng(5)
    x = np.concatenate([np.exp(rng.uniform(-40, 40, 200000)), rng.uniform(0, 3, 100000),
                        np.array([0.0, 1.0, 5e-324, 1e308, np.inf])])
    for y in (1 / 2.4, -1.4, -(0.4 / 2.8), 0.4 / 2.8, 2.8 / 0.4, 2.4, 1.4, (-1.4) * (1 / 2.4)):
        host = shared_pow(x, y)
        dev = np.empty_like(x)
        assert _lib.load().ef_pow_device(x.ctypes.data, y, dev.ctypes.data, x.size) == 0
        assert np.array_equal(host, dev, equal_nan=True)
        assert np.array_equal(host, O.shared_pow(x, y), equal_nan=True)


def test_perf_report_and_snapshot(tmp_path):  # perf.py:92-153, output.py:53-106
    from paper_2007_00094_b200 import output, perf

    ps = P.isentropic_vortex(24)
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    s.set_state(ps.U0)
    s.enable_timers(True)
    for _ in range(3):
        s.ssp_rk3_step()
    txt = perf.report(s, csv_path=str(tmp_path / "perf.csv"))
    assert "s/stage" in txt and "syncs=" in txt
    assert (tmp_path / "perf.csv").read_text().startswith("phase,kernel")
    output.write_vtk(str(tmp_path / "v.vtk"), ps.mesh, s.get_state(), ps.matrices)
    assert (tmp_path / "v.vtk").stat().st_size > 0


def test_graph_replay_is_bitwise_identical():
    """Steps replayed from captured CUDA graphs equal directly launched steps:
    RK3 and Euler, CFL and given tau, tau_max, the async chain, a state reset
    between replays, and the step counter."""
    ps = P.make_config("c1", scale="small")
    runs = []
    for graphs in (True, False):
        s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
        s.enable_graphs(graphs)
        s.set_state(ps.U0)
        taus = [s.ssp_rk3_step() for _ in range(4)]
        taus.append(s.euler_step(tau=1e-3))
        taus.append(s.euler_step(tau=1e-3))
        taus.append(s.euler_step(tau=5e-4))
        taus.append(s.ssp_rk3_step(tau_max=1e-3))
        mid = s.get_state()
        s.set_state(mid)
        for _ in range(5):
            s.ssp_rk3_step_async()
        taus.append(s.sync())
        runs.append((np.array(taus), s.get_state(), s.n_euler_steps))
    (ta, Ua, na), (tb, Ub, nb) = runs
    assert np.array_equal(ta, tb)
    assert np.array_equal(Ua, Ub)
    assert na == nb == 4 * 3 + 3 + 3 + 5 * 3


def test_stepping_after_an_error_restarts_from_the_kept_state():
    """After an AdmissibilityError the state is the one before the call, and
    the next steps equal those of a fresh solver from that state (nothing
    computed for the failed stages -- step0 fields, memo marks -- is reused)."""
    ps = P.make_config("c2", scale="small")
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    s.set_state(ps.U0)
    for _ in range(3):
        s.ssp_rk3_step()
    U = s.get_state()
    with pytest.raises(AdmissibilityError):
        s.euler_step(tau=5.0)  # far beyond the CFL bound
    assert np.array_equal(s.get_state(), U)
    taus = [s.ssp_rk3_step() for _ in range(3)]
    f = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    f.set_state(U)
    assert taus == [f.ssp_rk3_step() for _ in range(3)]
    assert np.array_equal(s.get_state(), f.get_state())


def test_async_chain_reports_an_error_of_a_middle_step():
    """Errors latch across a chain of async steps: a step in the middle of the
    chain that produces an inadmissible state is reported by sync(), even though
    the steps after it ran (and reset nothing).  The next set_state starts clean."""
    ps = P.make_config("c2", scale="small")
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    s.set_state(ps.U0)
    for _ in range(2):
        s.ssp_rk3_step()
    tau = s.tau_last
    U = s.get_state()
    s.ssp_rk3_step_async(tau=tau)
    s.ssp_rk3_step_async(tau=5.0)  # far beyond the CFL bound: inadmissible
    for _ in range(3):
        s.ssp_rk3_step_async(tau=tau)
    with pytest.raises(ValueError):  # AdmissibilityError (projection or bad state)
        s.sync()
    s.set_state(U)
    taus = [s.ssp_rk3_step() for _ in range(2)]
    f = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    f.set_state(U)
    assert taus == [f.ssp_rk3_step() for _ in range(2)]
    assert np.array_equal(s.get_state(), f.get_state())


def test_synchronous_calls_settle_a_pending_async_step():
    """ssp_rk3_step / euler_step / get_state after ssp_rk3_step_async continue
    from the async step's result (no step is lost or recomputed)."""
    ps = P.make_config("c1", scale="small")
    a = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    a.set_state(ps.U0)
    a.ssp_rk3_step_async()
    a.ssp_rk3_step()
    a.ssp_rk3_step_async()
    a.euler_step()
    a.ssp_rk3_step_async()
    Ua = a.get_state()
    b = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    b.set_state(ps.U0)
    b.ssp_rk3_step()
    b.ssp_rk3_step()
    b.ssp_rk3_step()
    b.euler_step()
    b.ssp_rk3_step()
    assert np.array_equal(Ua, b.get_state())
    assert a.n_euler_steps == b.n_euler_steps == 13


def test_advance_with_changing_tau_max_replays_one_graph():
    """advance() passes a different tau_max every step; tau and tau_max are
    kernel inputs in device memory, so graph replay stays bitwise identical to
    direct launches (and the captured graph is reused: one capture per key)."""
    ps = P.make_config("c1", scale="small")
    out = []
    for graphs in (True, False):
        s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
        s.enable_graphs(graphs)
        s.set_state(ps.U0)
        t = []
        s.advance(0.2, on_step=lambda k, tt: t.append(tt))
        out.append((t, s.get_state()))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])


def test_inadmissible_rk_step_reports_the_first_failing_stage_like_the_reference():
    """A step far beyond the CFL bound: the reference raises after the first stage
    whose result is inadmissible (stepper.py:612-622), naming its first bad
    node; the later stages (computed anyway on the device) must not change the
    reported error or node."""
    ps = P.make_config("c2", scale="small")
    s = Solver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    o = O.OracleSolver(ps.matrices, c_cfl=ps.c_cfl, boundary=ps.boundary)
    s.set_state(ps.U0)
    o.set_state(ps.U0)
    for _ in range(3):
        assert s.ssp_rk3_step() == o.ssp_rk3_step()
    for tau in (5.0, 0.5):
        with pytest.raises(ValueError) as eg:
            s.ssp_rk3_step(tau=tau)
        with pytest.raises(ValueError) as eo:
            o.ssp_rk3_step(tau)
        assert str(eg.value) == str(eo.value), tau
        o.set_state(s.get_state())

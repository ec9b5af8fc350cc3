"""Generate the golden parity fixtures from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --c1-full  # + C1 full size, 100 RK steps (~3 min)

The reference `eulerflow.stepper.Solver` (/root/reference/pkg/src) is imported
read-only and driven through its own public API.  The only configuration
change is the reference's own plug-in point for pow,
`physics.set_power_function` (physics.py:59-75), which is set to the host build
of the shared deterministic pow (paper_2007_00094_b200/csrc/ef_pow.h, exported
by the oracle library as `or_pow`).  Without that, numpy's SIMD pow (which
differs from libm on ~5% of inputs) makes bitwise parity impossible
(SURVEY.md §0, §8(c)).  A second, report-only record is made with numpy's
default pow for the divergence table in DESIGN.md.

Every fixture stores its inputs (PrecomputedMatrices, U0, boundary data,
parameters) and the reference outputs (tau per step, final state, and for the
first forward-Euler stage the internal arrays d, alpha, R, bounds, l mapped to
global Cuthill-McKee row order).  `/root/reference` does not exist on the GPU
box; the fixtures do.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, REPO)

from eulerflow import assembly as r_assembly  # noqa: E402
from eulerflow import mesh as r_mesh  # noqa: E402
from eulerflow import physics as r_physics  # noqa: E402
from eulerflow import problems as r_problems  # noqa: E402
from eulerflow import limiter as r_limiter  # noqa: E402
from eulerflow import riemann as r_riemann  # noqa: E402
from eulerflow.assembly import PrecomputedMatrices as RefMatrices  # noqa: E402
from eulerflow.stepper import BoundaryConditions as RefBC  # noqa: E402
from eulerflow.stepper import Solver as RefSolver  # noqa: E402

import oracle as O  # noqa: E402
from paper_2007_00094_b200 import problems as P  # noqa: E402


def to_ref_matrices(m) -> RefMatrices:
    return RefMatrices(n=int(m.n), dim=int(m.dim), indptr=np.asarray(m.indptr), indices=np.asarray(m.indices),
                       m=np.asarray(m.m), c=np.asarray(m.c), beta=np.asarray(m.beta),
                       m_lumped=np.asarray(m.m_lumped), inv_m=np.asarray(m.inv_m))


def to_ref_bc(bc):
    if bc is None:
        return None
    return RefBC(inflow_nodes=bc.inflow_nodes, farfield=bc.farfield,
                 slip_nodes=bc.slip_nodes, slip_normals=bc.slip_normals)


def internals_cm(solver: RefSolver):
    """First-stage internal arrays of rank 0, rows mapped to global CM order."""
    rk = solver.ranks[0]
    n_lo = rk.numbering.n_lo
    cm = rk.cm_of_new[:n_lo]
    out = {}
    for name in ("d", "l"):
        a = np.empty((solver.n, rk.width))
        a[cm] = getattr(rk, name)[:n_lo]
        out["int_" + name] = a
    a = np.empty((solver.n, rk.width, solver.nvar))
    a[cm] = rk.P[:n_lo]
    out["int_P"] = a
    a = np.empty(solver.n)
    a[cm] = rk.alpha[:n_lo]
    out["int_alpha"] = a
    a = np.empty((solver.n, solver.nvar))
    a[cm] = rk.R[:n_lo]
    out["int_R"] = a
    a = np.empty((solver.n, 3))
    a[cm, 0] = rk.rho_min[:n_lo]
    a[cm, 1] = rk.rho_max[:n_lo]
    a[cm, 2] = rk.phi_min[:n_lo]
    out["int_bounds"] = a
    return out


def run_reference(mat, U0, bc, params, steps, mode, record_internals=True):
    kw = dict(c_cfl=params["c_cfl"], limiter_passes=params["passes"], newton_steps=params["newton"])
    s = RefSolver(mat, boundary=bc, **kw)
    s.set_state(U0)
    taus = []
    out = {}
    for k in range(steps):
        if mode == "euler":
            taus.append(s.euler_step(params.get("tau")))
        else:
            taus.append(s.ssp_rk3_step(params.get("tau")))
        if k == 0 and record_internals and mode == "euler":
            out.update(internals_cm(s))
    out["taus"] = np.array(taus)
    out["U_final"] = s.get_state()
    return out


def save_case(name, mat, U0, bc, params, steps, mode, record_internals=True):
    res = run_reference(to_ref_matrices(mat), U0, to_ref_bc(bc), params, steps, mode, record_internals)
    rec = dict(
        n=np.int64(mat.n), dim=np.int64(mat.dim), indptr=np.asarray(mat.indptr, np.int64),
        indices=np.asarray(mat.indices, np.int32), m=np.asarray(mat.m), c=np.asarray(mat.c),
        m_lumped=np.asarray(mat.m_lumped), inv_m=np.asarray(mat.inv_m), U0=np.asarray(U0),
        params=json.dumps(dict(params, steps=steps, mode=mode)),
    )
    if bc is not None:
        if bc.inflow_nodes is not None:
            rec["bc_inflow"] = np.asarray(bc.inflow_nodes, np.int64)
            rec["bc_farfield"] = np.asarray(bc.farfield, np.float64)
        if bc.slip_nodes is not None:
            rec["bc_slip"] = np.asarray(bc.slip_nodes, np.int64)
            rec["bc_normals"] = np.asarray(bc.slip_normals, np.float64)
    rec.update(res)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"{name:28s} n={mat.n:6d} steps={steps} mode={mode} -> {os.path.getsize(path)/1024:.0f} KiB")


def ref_2d(meshobj):
    m = r_assembly.assemble(meshobj)
    return P.PrecomputedMatrices(n=m.n, dim=m.dim, indptr=m.indptr, indices=m.indices, m=m.m, c=m.c,
                                 beta=m.beta, m_lumped=m.m_lumped, inv_m=m.inv_m)


def base(c_cfl=0.9, passes=2, newton=2, tau=None):
    d = dict(c_cfl=c_cfl, passes=passes, newton=newton)
    if tau is not None:
        d["tau"] = tau
    return d


def small_cases():
    # reference test fixture: 4x4 periodic + default_rng(7) field (test_stepper.py:15-29)
    mat = ref_2d(r_mesh.rectangle_mesh(4, 4, periodic=(True, True)))
    U = P.random_state(np.random.default_rng(7), mat.n)
    for passes in (0, 1, 2, 3):
        save_case(f"periodic4_euler_p{passes}", mat, U, None, base(passes=passes), 1, "euler")
    save_case("periodic4_rk3", mat, U, None, base(), 4, "rk3")
    save_case("periodic4_newton4_p3", mat, U, None, base(passes=3, newton=4), 2, "rk3")
    save_case("periodic4_newton1", mat, U, None, base(newton=1), 2, "rk3")
    Uc = np.tile([1.4, 4.2, 0.0, 8.8], (mat.n, 1))
    save_case("periodic4_constant", mat, Uc, None, base(tau=1e-3), 1, "euler")
    # reference problems (problems.py) on reference meshes and assembly
    st = r_problems.mach3_channel(2, refine=2)
    save_case("mach3_channel_r2", ref_2d(st.mesh), st.U0, st.boundary, base(), 3, "rk3")
    save_case("mach3_channel_r2_euler", ref_2d(st.mesh), st.U0, st.boundary, base(), 1, "euler")
    st = r_problems.sod1d(60)
    save_case("sod1d_60", ref_2d(st.mesh), st.U0, None, base(), 8, "rk3")
    # BASELINE configs at oracle sizes, on this package's generators
    ps = P.isentropic_vortex(32)
    save_case("c1_vortex32", ps.matrices, ps.U0, ps.boundary, base(c_cfl=0.5), 5, "rk3")
    save_case("c1_vortex32_euler", ps.matrices, ps.U0, ps.boundary, base(c_cfl=0.5), 1, "euler")
    save_case("c1_vortex32_p0", ps.matrices, ps.U0, ps.boundary, base(c_cfl=0.5, passes=0), 5, "rk3")
    ps = P.mach3_disc(20, seed=11)
    save_case("c2_disc20", ps.matrices, ps.U0, ps.boundary, base(), 4, "rk3")
    ps = P.sod_box(11, 3, 3, seed=5)
    save_case("c3_sodbox", ps.matrices, ps.U0, ps.boundary, base(), 4, "rk3")
    save_case("c3_sodbox_euler", ps.matrices, ps.U0, ps.boundary, base(), 1, "euler")
    ps = P.periodic_fourier_box(6, seed=3)
    save_case("c5_periodic6", ps.matrices, ps.U0, None, base(), 3, "rk3")
    mat = P.assemble_q1(P.box_mesh(4, 4, 4, periodic=(True, True, True)))
    U = P.random_state(np.random.default_rng(4096), mat.n, dim=3)
    save_case("periodic3d_random_euler", mat, U, None, base(), 1, "euler")
    save_case("periodic3d_random_rk3", mat, U, None, base(), 2, "rk3")
    c4_case()
    function_cases()


def c4_case():
    """C4-shaped (extruded O-grid around a cylinder), oracle size."""
    ps = P.mach3_cylinder(10, 3, seed=13)
    save_case("c4_cylinder", ps.matrices, ps.U0, ps.boundary, base(), 2, "rk3", record_internals=False)


def function_cases():
    """riemann.d_ij_low and limiter.limiter_compute of the unmodified reference on
    seeded batches (function-level parity, like test_riemann.py / test_limiter.py):
    densities 1e-3..10, pressures 1e-4..1e4 (log-uniform), |u| ~ N(0, 2), equal
    states, equal pressures, zero and exactly antisymmetric c vectors; limiter
    lanes with corrections from 1e-2 to 10 times the state, bounds around it."""
    gas = r_physics.AIR
    for dim in (2, 3):
        rng = np.random.default_rng(7000 + dim)
        n = 3000

        def states(k):
            rho = np.exp(rng.uniform(np.log(1e-3), np.log(10.0), k))
            u = rng.normal(0.0, 2.0, (k, dim))
            p = np.exp(rng.uniform(np.log(1e-4), np.log(1e4), k))
            U = np.empty((k, dim + 2))
            U[:, 0] = rho
            U[:, 1:-1] = rho[:, None] * u
            U[:, -1] = p / gas.gm1 + 0.5 * rho * (u * u).sum(axis=1)
            return U

        Ui, Uj = states(n), states(n)
        Uj[: n // 10] = Ui[: n // 10]                               # identical pairs
        k = slice(n // 10, n // 5)                                     # equal pressures
        pi = gas.gm1 * (Ui[k, -1] - 0.5 * (Ui[k, 1:-1] ** 2).sum(axis=1) / Ui[k, 0])
        Uj[k, -1] = pi / gas.gm1 + 0.5 * (Uj[k, 1:-1] ** 2).sum(axis=1) / Uj[k, 0]
        cij = rng.normal(0.0, 1.0, (n, dim))
        cji = rng.normal(0.0, 1.0, (n, dim))
        cji[n // 5: n // 2] = -cij[n // 5: n // 2]                     # antisymmetric
        cij[-n // 20:] = 0.0                                           # zero c_ij
        cji[-n // 40:] = 0.0
        d = r_riemann.d_ij_low(Ui, Uj, cij, cji, gas)
        U = states(n)
        scale = np.exp(rng.uniform(np.log(1e-2), np.log(10.0), n))
        Pc = rng.normal(0.0, 1.0, (n, dim + 2)) * U * scale[:, None]
        rho = U[:, 0]
        rmin = rho * (1.0 - rng.uniform(0.0, 0.3, n))
        rmax = rho * (1.0 + rng.uniform(0.0, 0.3, n))
        eps = U[:, -1] - 0.5 * (U[:, 1:-1] ** 2).sum(axis=1) / rho
        phi = eps * rho ** (-gas.gamma)
        pmin = phi * (1.0 - rng.uniform(0.0, 0.1, n))
        pmin[: n // 10] = phi[: n // 10]                               # bound at the state itself
        bounds = np.column_stack([rmin, rmax, pmin])
        l2 = r_limiter.limiter_compute(U, Pc, rmin, rmax, pmin, 2, gas)
        l4 = r_limiter.limiter_compute(U, Pc, rmin, rmax, pmin, 4, gas)
        path = os.path.join(HERE, f"functions_{dim}d.npz")
        np.savez_compressed(path, Ui=Ui, Uj=Uj, cij=cij, cji=cji, d=d, U=U, P=Pc, bounds=bounds,
                            l_newton2=l2, l_newton4=l4)
        print(f"functions_{dim}d: d in [{d.min():.3g}, {d.max():.3g}], "
              f"l<1 on {int((l2 < 1).sum())}/{n} lanes -> {os.path.getsize(path) / 1024:.0f} KiB")


def c1_full():
    """C1 at full size (129x129, CFL 0.5, 100 RK steps).  Too large to commit
    with its inputs, so the fixture holds digests: the test regenerates the
    inputs with this package's generator, checks their digest, runs the oracle
    and compares the output digest + a few norms."""
    ps = P.isentropic_vortex(128)
    mat = ps.matrices
    h_in = hashlib.sha256()
    for a in (mat.indptr, mat.indices, mat.m, mat.c, mat.m_lumped, mat.inv_m, ps.U0,
              ps.boundary.inflow_nodes, ps.boundary.farfield):
        h_in.update(np.ascontiguousarray(a).tobytes())
    res = run_reference(to_ref_matrices(mat), ps.U0, to_ref_bc(ps.boundary), base(c_cfl=0.5), 100,
                        "rk3", record_internals=False)
    U = res["U_final"]
    rec = dict(input_sha256=h_in.hexdigest(),
               output_sha256=hashlib.sha256(np.ascontiguousarray(U).tobytes()).hexdigest(),
               taus=res["taus"].tolist(), min_rho=float(U[:, 0].min()),
               sum_state=np.asarray(U.sum(axis=0)).tolist(), n=int(mat.n), steps=100, c_cfl=0.5)
    with open(os.path.join(HERE, "c1_full_100.json"), "w") as fh:
        json.dump(rec, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "c1_full_100_state.npz"), U_final=U)
    print("c1_full_100", rec["output_sha256"], rec["min_rho"])


def input_digest(mat, U0, bc) -> str:
    """sha256 over the inputs in a fixed order (tests/stated.py recomputes it)."""
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


# BASELINE configs at the step counts BASELINE.json states, at the sizes the
# reference finishes in minutes here (SURVEY.md §8(c) "Recommended" column).
# Generator calls are this package's (problems.py), default seeds.
STATED = {
    "c2_full_20": dict(gen="mach3_disc", args=(550,), steps=20, every=5,
                       note="C2 at full size (1.23M nodes), 20-step prefix of the 200"),
    "c3_128x32x32_100": dict(gen="sod_box", args=(127, 31, 31), steps=100, every=10,
                             note="C3 Sod box at 128x32x32 nodes (jittered), 100 steps (stated)"),
    "c4_210k_50": dict(gen="mach3_cylinder", args=(40, 30), steps=50, every=10,
                       note="C4 extruded O-grid at 0.21M nodes, 50 steps (stated)"),
    "c5_64_50": dict(gen="periodic_fourier_box", args=(64,), steps=50, every=10,
                     note="C5 periodic Fourier box at 64^3, 50 steps (stated)"),
}


def stated_case(name, workers):
    """Run the UNMODIFIED reference Solver for the stated number of SSP-RK3 steps
    and record digests: input sha256, tau of every step, sha256 of U every
    `every` steps and at the end, plus norms.  The GPU test and the oracle test
    regenerate the inputs with problems.py, check the input digest and compare
    their own digests bit for bit (tests/test_gpu_stated.py)."""
    import time
    spec = STATED[name]
    ps = getattr(P, spec["gen"])(*spec["args"])
    mat = ps.matrices
    t0 = time.time()
    s = RefSolver(to_ref_matrices(mat), boundary=to_ref_bc(ps.boundary), c_cfl=ps.c_cfl,
                  limiter_passes=2, newton_steps=2, workers=workers)
    s.set_state(ps.U0)
    t_setup = time.time() - t0
    taus, digests = [], {}
    t0 = time.time()
    for k in range(1, spec["steps"] + 1):
        taus.append(s.ssp_rk3_step())
        if k % spec["every"] == 0 or k == spec["steps"]:
            U = s.get_state()
            digests[str(k)] = state_digest(U)
            print(f"  {name} step {k}: {digests[str(k)][:16]} ({time.time() - t0:.0f} s)", flush=True)
    U = s.get_state()
    rec = dict(config=name, note=spec["note"], generator=spec["gen"], args=list(spec["args"]),
               n=int(mat.n), nnz=int(mat.nnz), dim=int(mat.dim), c_cfl=ps.c_cfl, limiter_passes=2,
               newton_steps=2, steps=spec["steps"], input_sha256=input_digest(mat, ps.U0, ps.boundary),
               taus=taus, state_sha256=digests, min_rho=float(U[:, 0].min()),
               sum_state=np.asarray(U.sum(axis=0)).tolist(),
               reference=dict(workers=workers, setup_s=round(t_setup, 1),
                              steps_s=round(time.time() - t0, 1), numpy=np.__version__))
    with open(os.path.join(HERE, f"stated_{name}.json"), "w") as fh:
        json.dump(rec, fh, indent=1)
    print(name, "done", rec["reference"], flush=True)


def default_pow_divergence():
    """Report-only: reference with numpy's default pow vs the shared pow."""
    ps = P.isentropic_vortex(32)
    out = {}
    for steps in (1, 5, 20):
        r_physics.set_power_function(O.shared_pow)
        a = run_reference(to_ref_matrices(ps.matrices), ps.U0, to_ref_bc(ps.boundary), base(c_cfl=0.5),
                          steps, "rk3", False)["U_final"]
        r_physics.set_power_function(None)
        b = run_reference(to_ref_matrices(ps.matrices), ps.U0, to_ref_bc(ps.boundary), base(c_cfl=0.5),
                          steps, "rk3", False)["U_final"]
        out[steps] = float(np.abs(a - b).max() / np.abs(b).max())
    r_physics.set_power_function(O.shared_pow)
    with open(os.path.join(HERE, "default_pow_divergence.json"), "w") as fh:
        json.dump({"case": "c1_vortex32 rk3, rel Linf shared-pow vs numpy-pow reference", "rel_linf": out,
                   "numpy": np.__version__}, fh, indent=1)
    print("default-pow divergence", out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1-full", action="store_true")
    ap.add_argument("--only-c1-full", action="store_true")
    ap.add_argument("--only-c4", action="store_true")
    ap.add_argument("--only-functions", action="store_true")
    ap.add_argument("--stated", nargs="*", metavar="CASE",
                    help=f"reference digests at the stated step counts: {', '.join(STATED)}")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    r_physics.set_power_function(O.shared_pow)
    if args.stated is not None:
        for name in args.stated or list(STATED):
            stated_case(name, args.workers)
    elif args.only_c4:
        c4_case()
    elif args.only_functions:
        function_cases()
    elif not args.only_c1_full:
        small_cases()
        default_pow_divergence()
    if args.c1_full or args.only_c1_full:
        c1_full()

"""`Solver`: the reference's time-integrator API over the B200 C-ABI.

Drop-in for `eulerflow.stepper.Solver` (/root/reference/pkg/src/eulerflow/
stepper.py:87-649): same constructor signature, same methods (set_state,
get_state, euler_step, ssp_rk3_step, advance), same attributes (tau_last,
timers, n_euler_steps, standard_card, comm.sync_count/sync_volume) and the
same exceptions (ValueError, AdmissibilityError, RuntimeError).  Every stage
runs as hand-written sm_100a kernels inside libef_b200.so; this module only
computes the global Cuthill-McKee order (scipy, exactly as
exchange.partition does, exchange.py:58-62) and marshals arrays.

`lanes`, `workers` and `chunk_size` are accepted for signature
compatibility; the reference's results are bitwise independent of them
(test_stepper.py:106-128) and so are ours.  `overlap` (with ranks > 1)
computes the exported rows first and moves their halo on a second stream
while the interior rows are computed (exchange.py:168-222); results are
identical either way.  `ranks` > 1 partitions the mesh
into contiguous Cuthill-McKee ranges with ghost layers exactly like the
reference's simulated ranks (exchange.py:52-104) and steps them in lockstep
on one device; one process per GPU with NCCL is
paper_2007_00094_b200.distributed.DistributedSolver.
"""

from __future__ import annotations

import ctypes
from types import SimpleNamespace
from typing import Dict, Optional

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

from . import _lib
from .physics import AIR, AdmissibilityError, GasConstants, is_admissible
from .problems import BoundaryConditions

__all__ = ["Solver", "BoundaryConditions", "compute_tau", "cm_permutation", "STEP_NAMES", "eval_dij",
           "eval_limiter", "eval_arith"]

STEP_NAMES = ["step0", "step1", "step2", "step3", "step4", "step5", "step6"]


def compute_tau(d_diag: np.ndarray, m_i: np.ndarray, c_cfl: float) -> float:
    """CFL time step c_cfl * min_i m_i / (-2 d_ii) (stepper.py:55-63)."""
    mask = d_diag < 0.0
    if not mask.any():
        raise ValueError("constant field, the time step bound is unbounded")
    return c_cfl * float(np.min(m_i[mask] / (-2.0 * d_diag[mask])))


def cm_permutation(matrices):
    """Global Cuthill-McKee order of exchange.partition (exchange.py:58-62):
    returns (cm_perm: original -> CM id, cm_inv: CM id -> original)."""
    n = int(matrices.n)
    conn = sp.csr_matrix(
        (np.ones(len(matrices.indices), dtype=np.int8), np.asarray(matrices.indices),
         np.asarray(matrices.indptr)), shape=(n, n))
    sym = (conn + conn.T).tocsr()
    rcm = reverse_cuthill_mckee(sym, symmetric_mode=True)
    cm_inv = np.asarray(rcm[::-1], dtype=np.int64)
    cm_perm = np.empty(n, dtype=np.int64)
    cm_perm[cm_inv] = np.arange(n)
    return cm_perm, cm_inv


def _raise(code: int, msg: Optional[str] = None):
    if code == _lib.EF_OK:
        return
    if msg is None:
        msg = _lib.last_error()
    if code == _lib.EF_ERR_ARG:
        raise ValueError(msg)
    if code == _lib.EF_ERR_INADMISSIBLE:
        raise AdmissibilityError(msg)
    if code == _lib.EF_ERR_TAU_UNBOUNDED:
        raise ValueError(msg)
    raise RuntimeError(msg)


class Solver:
    """SSP-RK3 / forward-Euler IDP stage on one B200 (one rank per process)."""

    def __init__(self, matrices, c_cfl: float = 0.9, limiter_passes: int = 2, newton_steps: int = 2,
                 lanes: int = 4, workers: int = 1, ranks: int = 1, overlap: bool = True,
                 chunk_size: int = 2048, boundary: Optional[BoundaryConditions] = None,
                 gas: GasConstants = AIR, device: int = 0, stream=None,
                 cm_perm: Optional[np.ndarray] = None, ranges=None, nccl_rank=None):
        if not 0.0 < c_cfl <= 1.0:
            raise ValueError("c_cfl must lie in (0, 1]")
        if limiter_passes < 0:
            raise ValueError("limiter_passes must be >= 0")
        self.matrices = matrices
        self.gas = gas
        self.c_cfl = c_cfl
        self.limiter_passes = limiter_passes
        self.newton_steps = newton_steps
        self.lanes, self.workers, self.overlap, self.chunk_size = lanes, workers, overlap, chunk_size
        self.bc = boundary
        self.n = int(matrices.n)
        self.dim = int(matrices.dim)
        self.nvar = self.dim + 2
        self.ranks = ranks
        lib = _lib.load()
        if cm_perm is None:
            cm_perm, cm_inv = cm_permutation(matrices)
        else:
            cm_perm = np.asarray(cm_perm, dtype=np.int64)
            cm_inv = np.empty_like(cm_perm)
            cm_inv[cm_perm] = np.arange(self.n)
        self.cm_perm, self.cm_inv = cm_perm, cm_inv
        keep = []

        def ptr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data

        mats = _lib.EfMatrices(
            self.n, self.dim, ptr(matrices.indptr, np.int64), ptr(matrices.indices, np.int64),
            ptr(matrices.m, np.float64), ptr(matrices.c, np.float64),
            ptr(matrices.m_lumped, np.float64), ptr(matrices.inv_m, np.float64))
        prm = _lib.EfParams(gas.gamma, gas.gm1, gas.gp1_inv, gas.gm1_over_2g, gas.two_g_over_gm1,
                            float(c_cfl), int(limiter_passes), int(newton_steps), int(bool(overlap)))
        bcs = _lib.EfBoundary(0, None, None, 0, None, None)
        if boundary is not None:
            if boundary.inflow_nodes is not None and len(boundary.inflow_nodes):
                bcs.n_inflow = len(boundary.inflow_nodes)
                bcs.inflow = ptr(boundary.inflow_nodes, np.int64)
                bcs.farfield = ptr(boundary.farfield, np.float64)
            if boundary.slip_nodes is not None and len(boundary.slip_nodes):
                bcs.n_slip = len(boundary.slip_nodes)
                bcs.slip = ptr(boundary.slip_nodes, np.int64)
                bcs.slip_normals = ptr(boundary.slip_normals, np.float64)
        if stream is not None:
            stream = int(stream)
            if stream == 0:  # the legacy default stream (torch's default) is handle 1
                stream = 1
        ranges = None if ranges is None else ptr(np.asarray(ranges, dtype=np.int64), np.int64)
        self._handles = []
        self._group = None
        if nccl_rank is not None:
            # one rank of a one-process-per-GPU NCCL job (paper_2007_00094_b200.distributed)
            r, R, uid = nccl_rank
            idbuf = ctypes.create_string_buffer(bytes(uid), 128)
            keep.append(idbuf)
            specs = [(int(r), int(R), ctypes.cast(idbuf, ctypes.c_void_p).value)]
        else:
            # ranks > 1: the reference's simulated ranks as a same-device group
            R = max(1, int(ranks or 1))
            specs = [(r, R, None) for r in range(R)]
        for r, R, uid in specs:
            dist = _lib.EfDist(r, R, int(device), ptr(cm_perm, np.int64), ranges, uid, stream)
            h = ctypes.c_void_p()
            rc = lib.ef_create(ctypes.byref(mats), ctypes.byref(prm), ctypes.byref(bcs),
                               ctypes.byref(dist), ctypes.byref(h))
            if rc != _lib.EF_OK:
                msg = _lib.last_error()
                self.close()
                _raise(rc, msg)
            self._handles.append(h)
        if nccl_rank is None and len(self._handles) > 1:
            arr = (ctypes.c_void_p * len(self._handles))(*[h.value for h in self._handles])
            g = ctypes.c_void_p()
            _raise(lib.ef_group_create(arr, len(self._handles), ctypes.byref(g)))
            self._group = g
        self._h = self._handles[0]
        del keep
        info = np.zeros(6, dtype=np.int64)
        lib.ef_info(self._h, info.ctypes.data)
        self.n_owned, self.n_local, self.pad_width, self.nnz_owned, self.standard_card = (
            int(x) for x in info[:5])
        self.n_euler_steps = 0
        self.tau_last = None
        self._timers_on = False

    @property
    def comm(self):
        """sync_count / sync_volume of the halo exchanges (exchange.py:131-157)."""
        tot = np.zeros(3, dtype=np.int64)
        for h in self._handles:
            c = np.zeros(3, dtype=np.int64)
            _lib.load().ef_counters(h, c.ctypes.data)
            tot[2] += c[2]
            tot[1] = c[1]
        return SimpleNamespace(sync_count=int(tot[1]), sync_volume=int(tot[2]))

    # ----- lifecycle ------------------------------------------------------
    def close(self):
        lib = _lib.load()
        g = getattr(self, "_group", None)
        if g:
            lib.ef_group_destroy(g)
            self._group = None
        for h in reversed(getattr(self, "_handles", [])):  # rank 0 owns a group's stream: last
            if h:
                lib.ef_destroy(h)
        self._handles = []
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----- state ----------------------------------------------------------
    def set_state(self, U: np.ndarray):
        """Load states given in original node order (stepper.py:319-328)."""
        U = np.ascontiguousarray(U, dtype=np.float64)
        if U.shape != (self.n, self.nvar):
            raise ValueError("state array has the wrong shape")
        lib = _lib.load()
        rc = (lib.ef_group_set_state(self._group, U.ctypes.data) if self._group
              else lib.ef_set_state(self._h, U.ctypes.data))
        if rc == _lib.EF_ERR_INADMISSIBLE:
            raise AdmissibilityError("initial state is not admissible")
        _raise(rc)

    def get_state(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """States in original node order (stepper.py:330-336); on an NCCL rank
        only the owned rows are filled (see distributed.DistributedSolver)."""
        if out is None:
            out = np.zeros((self.n, self.nvar))
        lib = _lib.load()
        _raise(lib.ef_group_get_state(self._group, out.ctypes.data) if self._group
               else lib.ef_get_state(self._h, out.ctypes.data))
        return out

    # ----- stepping -------------------------------------------------------
    def euler_step(self, tau: Optional[float] = None, tau_max: float = np.inf) -> float:
        t = ctypes.c_double()
        lib = _lib.load()
        args = (0 if tau is None else 1, 0.0 if tau is None else float(tau), float(tau_max), ctypes.byref(t))
        rc = lib.ef_group_euler_step(self._group, *args) if self._group else lib.ef_euler_step(self._h, *args)
        _raise(rc)
        self.tau_last = t.value
        self.n_euler_steps += 1
        return t.value

    def ssp_rk3_step(self, tau: Optional[float] = None, tau_max: float = np.inf) -> float:
        t = ctypes.c_double()
        lib = _lib.load()
        args = (0 if tau is None else 1, 0.0 if tau is None else float(tau), float(tau_max), ctypes.byref(t))
        rc = lib.ef_group_ssp_rk3_step(self._group, *args) if self._group else lib.ef_ssp_rk3_step(self._h, *args)
        _raise(rc)
        self.tau_last = t.value
        self.n_euler_steps += 3
        return t.value

    def ssp_rk3_step_async(self, tau: Optional[float] = None, tau_max: float = np.inf):
        """Enqueue one RK step without a host sync; errors surface at sync()."""
        rc = _lib.load().ef_ssp_rk3_step_async(self._h, 0 if tau is None else 1,
                                               0.0 if tau is None else float(tau), float(tau_max))
        _raise(rc)
        self.n_euler_steps += 3

    def sync(self) -> float:
        t = ctypes.c_double()
        _raise(_lib.load().ef_sync(self._h, ctypes.byref(t)))
        self.tau_last = t.value
        return t.value

    def advance(self, t_final: float, use_rk3: bool = True, on_step=None) -> int:
        """March from t = 0 to t_final (stepper.py:638-649)."""
        t = 0.0
        steps = 0
        while t < t_final - 1e-14:
            step = self.ssp_rk3_step if use_rk3 else self.euler_step
            tau = step(tau_max=t_final - t)
            t += tau
            steps += 1
            if on_step is not None:
                on_step(steps, t)
        return steps

    # ----- observability --------------------------------------------------
    def enable_timers(self, on: bool = True):
        _raise(_lib.load().ef_enable_timers(self._h, 1 if on else 0))
        self._timers_on = on

    def enable_graphs(self, on: bool = True):
        """CUDA-graph replay of whole steps (default on; identical results)."""
        for h in self._handles:
            _raise(_lib.load().ef_enable_graphs(h, 1 if on else 0))

    def set_uniform_shortcuts(self, mode: int = -1):
        """Identical-state shortcuts: -1 automatic (default), 0 off, 1 on; identical results."""
        for h in self._handles:
            _raise(_lib.load().ef_set_uniform(h, int(mode)))

    @property
    def timers(self) -> Dict[str, float]:
        s = np.zeros(7)
        _lib.load().ef_phase_times(self._h, s.ctypes.data)
        return {name: float(v) for name, v in zip(STEP_NAMES, s)}

    _FIELDS = {"d": 0, "alpha": 1, "R": 2, "bounds": 3, "l": 4, "eor": 5, "phi": 6, "U": 7, "U_next": 8,
               "l_prev": 9, "P_stored": 10}

    def fetch(self, which: str, pass_index: int = 0) -> np.ndarray:
        """Internal arrays of the last stage (rows = local rows in global CM order; slots
        in stencil order), the reference's rk.* arrays (stepper.py:73-84, 456-491):
        "d", "alpha", "R", "bounds" (rho_min, rho_max, phi_min), "U_next", "eor", "phi";
        "P": rk.P after the stage, i.e. the correction fluxes the last limiter pass
        used: P_0 (1 - min l_0) ... (1 - min l_{q-1}) (stepper.py:468, 485);
        "l" / "l_prev": min(l_ij, l_ji) of the last / the previous pass.  The last pass
        runs only on the edges whose previous factor was below 1 (elsewhere its P is
        +-0 and the factor does not enter the result): "l" holds its value there and an
        earlier value elsewhere.  Slots of edges on the exact P = 0 fast path
        (identical-state mode) hold the tag -1 in "l_prev"; their "P" is a zero whose
        sign is not tracked."""
        n, L, nv = self.n_local, self.pad_width, self.nvar
        if which == "P":
            if self.limiter_passes == 0:
                return np.zeros((n, L, nv))
            P = self.fetch("P_stored")
            if self.limiter_passes == 1:
                return P
            ml = self.fetch("l_prev")
            fac = np.where(ml < 0.0, 0.0, 1.0 - ml)
            return P * fac[..., None]
        shapes = {"d": (n, L), "alpha": (n,), "R": (n, nv), "bounds": (n, 3), "l": (n, L),
                  "eor": (n,), "phi": (n,), "U": (n, nv), "U_next": (n, nv), "l_prev": (n, L),
                  "P_stored": (n, L, nv)}
        out = np.empty(shapes[which])
        _raise(_lib.load().ef_debug_fetch(self._h, self._FIELDS[which], int(pass_index), out.ctypes.data))
        return out

    def local_gids(self) -> np.ndarray:
        out = np.empty(self.n_local, dtype=np.int64)
        _raise(_lib.load().ef_local_gids(self._h, out.ctypes.data))
        return out


def shared_pow(x, y):
    """Host build of the device pow (ef_pow_host), numpy.power calling convention;
    install into the reference with physics.set_power_function(shared_pow)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    yv = np.asarray(y, dtype=np.float64)
    out = np.empty_like(x)
    if yv.ndim == 0:
        _lib.load().ef_pow_host(x.ctypes.data, float(yv), out.ctypes.data, x.size)
    else:
        xb, yb = np.broadcast_arrays(x, yv)
        out = np.empty(xb.shape)
        flat_x = np.ascontiguousarray(xb).ravel()
        flat_y = np.ascontiguousarray(yb).ravel()
        o = out.reshape(-1)
        for k in range(flat_x.size):
            tmp = np.empty(1)
            _lib.load().ef_pow_host(flat_x[k:k + 1].ctypes.data, float(flat_y[k]), tmp.ctypes.data, 1)
            o[k] = tmp[0]
    return out if out.ndim else out[()]


def _params(gas, newton_steps=2):
    gas = gas if gas is not None else AIR
    return _lib.EfParams(gas.gamma, gas.gm1, gas.gp1_inv, gas.gm1_over_2g, gas.two_g_over_gm1,
                         0.9, 2, int(newton_steps), 1)


def eval_dij(Ui, Uj, cij, cji, gas=None):
    """riemann.d_ij_low (riemann.py:119-142) on a batch of independent pairs,
    evaluated on the GPU by the stage's own device code.  Returns (d, bad) with
    bad = projection error flags (rho <= 0 or p <= 0)."""
    Ui, Uj, cij, cji = (np.ascontiguousarray(a, dtype=np.float64) for a in (Ui, Uj, cij, cji))
    n, dim = cij.shape
    out = np.empty(n)
    bad = np.zeros(n, dtype=np.int32)
    prm = _params(gas)
    _raise(_lib.load().ef_eval_dij(ctypes.byref(prm), dim, n, Ui.ctypes.data, Uj.ctypes.data,
                                   cij.ctypes.data, cji.ctypes.data, out.ctypes.data, bad.ctypes.data))
    return out, bad


def eval_limiter(U, P, bounds, newton_steps=2, gas=None):
    """limiter.limiter_compute (limiter.py:149-193) lane by lane on the GPU;
    bounds = (n, 3) rho_min, rho_max, phi_min."""
    U, P, bounds = (np.ascontiguousarray(a, dtype=np.float64) for a in (U, P, bounds))
    n, nv = U.shape
    out = np.empty(n)
    prm = _params(gas, newton_steps)
    _raise(_lib.load().ef_eval_limiter(ctypes.byref(prm), nv - 2, n, U.ctypes.data, P.ctypes.data,
                                       bounds.ctypes.data, out.ctypes.data))
    return out


def eval_arith(a, b):
    """Mismatch counts of the d_ij kernel's straight-line 1/b, a/b, sqrt|a| and shared-reciprocal
    a/b (csrc/ef_math.cuh) against the IEEE operations, over the operands inside the safe range."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape or a.ndim != 1:
        raise ValueError("a and b must be 1-D arrays of one length")
    out = np.zeros(4, dtype=np.uint64)
    _raise(_lib.load().ef_eval_arith(a.size, a.ctypes.data, b.ctypes.data, out.ctypes.data))
    return out

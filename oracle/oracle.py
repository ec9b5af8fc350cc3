"""ctypes front-end of the CPU oracle (idp_oracle.c).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product.

`OracleSolver` mirrors the reference `Solver` API
(/root/reference/pkg/src/eulerflow/stepper.py:87-649) for a single rank.  Its
setup restates the reference's global ordering independently of the product:
the Cuthill-McKee permutation of `exchange.partition` (exchange.py:58-62),
the CM-permuted CSR of `Solver._permute_matrices` (stepper.py:143-161) and the
global pad width (stepper.py:128-131).  Slot order inside a row is ascending
CM id (stepper.py:195), which fixes every floating-point reduction order.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libidp_oracle.so")
_lib = None

OR_OK, OR_ADMISSIBILITY, OR_BAD_STATE, OR_TAU_UNBOUNDED = 0, 1, 2, 3

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_d = ctypes.c_double
_i = ctypes.c_int


class AdmissibilityError(ValueError):
    pass


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_create.restype = _p
        L.or_create.argtypes = [_i64, _i, _i, _p, _p, _p, _p, _p, _p, _p, _d, _i, _i,
                                _i64, _p, _p, _i64, _p, _p, _i]
        L.or_destroy.argtypes = [_p]
        L.or_set_state.argtypes = [_p, _p]
        L.or_get_state.argtypes = [_p, _p]
        L.or_euler_step.argtypes = [_p, _i, _d, _d, _p]
        L.or_euler_step.restype = _i
        L.or_ssp_rk3_step.argtypes = [_p, _i, _d, _d, _p]
        L.or_ssp_rk3_step.restype = _i
        L.or_bad_row.argtypes = [_p]
        L.or_bad_row.restype = _i64
        L.or_fetch.argtypes = [_p, _i, _p]
        L.or_fetch.restype = _i
        L.or_set_threads.argtypes = [_p, _i]
        L.or_pow.argtypes = [_p, _d, _p, _i64]
        L.or_pow2.argtypes = [_p, _p, _p, _i64]
        L.or_eval_dij.argtypes = [_i, _d, _d, _d, _d, _d, _i64, _p, _p, _p, _p, _p, _p]
        L.or_eval_limiter.argtypes = [_i, _d, _d, _d, _d, _d, _i64, _p, _p, _p, _i, _p]
        _lib = L
    return _lib


def shared_pow(x, y):
    """Host build of ef_pow.h with numpy.power's calling convention; the
    function installed into the reference via physics.set_power_function."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    xb, yb = np.broadcast_arrays(x, y)
    xc = np.ascontiguousarray(xb)
    out = np.empty(xc.shape, dtype=np.float64)
    if y.ndim == 0:
        lib().or_pow(xc.ctypes.data, float(y), out.ctypes.data, xc.size)
    else:
        yc = np.ascontiguousarray(yb)
        lib().or_pow2(xc.ctypes.data, yc.ctypes.data, out.ctypes.data, xc.size)
    return out if out.ndim else out[()]


def cm_permutation(matrices):
    """Global Cuthill-McKee order exactly as exchange.partition (exchange.py:58-62)."""
    n = matrices.n
    conn = sp.csr_matrix(
        (np.ones(len(matrices.indices), dtype=np.int8), matrices.indices, matrices.indptr),
        shape=(n, n),
    )
    sym = (conn + conn.T).tocsr()
    rcm = reverse_cuthill_mckee(sym, symmetric_mode=True)
    cm_inv = np.asarray(rcm[::-1], dtype=np.int64)
    cm_perm = np.empty(n, dtype=np.int64)
    cm_perm[cm_inv] = np.arange(n)
    return cm_perm, cm_inv


class OracleSolver:
    """Single-rank CPU restatement of the reference Solver (test infrastructure)."""

    def __init__(self, matrices, c_cfl=0.9, limiter_passes=2, newton_steps=2,
                 boundary=None, gas=None, threads=1, cm_perm=None):
        """cm_perm: original id -> global order id replacing the Cuthill-McKee order
        (the per-rank setup's generator order, e.g. a box's lexicographic order);
        slots are sorted by it like the reference sorts them by CM id."""
        if not 0.0 < c_cfl <= 1.0:
            raise ValueError("c_cfl must lie in (0, 1]")
        if limiter_passes < 0:
            raise ValueError("limiter_passes must be >= 0")
        if gas is None:
            from types import SimpleNamespace
            g = 7.0 / 5.0
            gas = SimpleNamespace(gamma=g, gm1=g - 1.0, gp1_inv=1.0 / (g + 1.0),
                                  gm1_over_2g=(g - 1.0) / (2.0 * g), two_g_over_gm1=2.0 * g / (g - 1.0))
        self.n = int(matrices.n)
        self.dim = int(matrices.dim)
        self.nvar = self.dim + 2
        n, d = self.n, self.dim
        if cm_perm is None:
            self.cm_perm, self.cm_inv = cm_permutation(matrices)
        else:
            self.cm_perm = np.asarray(cm_perm, dtype=np.int64)
            self.cm_inv = np.empty_like(self.cm_perm)
            self.cm_inv[self.cm_perm] = np.arange(n)
        indptr = np.asarray(matrices.indptr, dtype=np.int64)
        indices = np.asarray(matrices.indices, dtype=np.int64)
        card_o = np.diff(indptr)
        row_o = np.repeat(np.arange(n), card_o)
        key = self.cm_perm[row_o] * n + self.cm_perm[indices]
        order = np.argsort(key, kind="stable")
        rows_cm = self.cm_perm[row_o][order]
        cols_cm = self.cm_perm[indices][order]
        card = np.bincount(rows_cm, minlength=n).astype(np.int64)
        L = int(card.max())
        self.width = L
        starts = np.concatenate([[0], np.cumsum(card)[:-1]])
        slot = np.arange(len(order)) - starts[rows_cm]
        pos = rows_cm * L + slot
        cols = np.repeat(np.arange(n, dtype=np.int64), L)
        cols[pos] = cols_cm
        c = np.zeros((n * L, d))
        c[pos] = np.asarray(matrices.c)[order]
        m_slot = np.zeros(n * L)
        m_slot[pos] = np.asarray(matrices.m)[order]
        m_i = np.ascontiguousarray(np.asarray(matrices.m_lumped)[self.cm_inv])
        inv_m = np.ascontiguousarray(np.asarray(matrices.inv_m)[self.cm_inv])
        gas5 = np.array([gas.gamma, gas.gm1, gas.gp1_inv, gas.gm1_over_2g, gas.two_g_over_gm1])
        self._keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a.ctypes.data

        inflow = np.zeros(0, dtype=np.int64)
        farfield = np.zeros(self.nvar)
        slip = np.zeros(0, dtype=np.int64)
        slip_n = np.zeros((0, d))
        if boundary is not None:
            if boundary.inflow_nodes is not None and len(boundary.inflow_nodes):
                inflow = self.cm_perm[np.asarray(boundary.inflow_nodes, dtype=np.int64)]
                farfield = np.asarray(boundary.farfield, dtype=np.float64)
            if boundary.slip_nodes is not None and len(boundary.slip_nodes):
                slip = self.cm_perm[np.asarray(boundary.slip_nodes, dtype=np.int64)]
                slip_n = np.asarray(boundary.slip_normals, dtype=np.float64)
        self._h = lib().or_create(
            n, d, L, arr(cols, np.int64), arr(card, np.int64), arr(c, np.float64),
            arr(m_slot, np.float64), arr(m_i, np.float64), arr(inv_m, np.float64),
            arr(gas5, np.float64), float(c_cfl), int(limiter_passes), int(newton_steps),
            len(inflow), arr(inflow, np.int64), arr(farfield, np.float64),
            len(slip), arr(slip, np.int64), arr(slip_n, np.float64), int(threads))
        self._keep = []
        if not self._h:
            raise ValueError("stencil pattern is not structurally symmetric")
        self.tau_last = None
        self.n_euler_steps = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().or_destroy(h)
            self._h = None

    def set_threads(self, threads: int):
        lib().or_set_threads(self._h, int(threads))

    def set_state(self, U):
        U = np.asarray(U, dtype=np.float64)
        if U.shape != (self.n, self.nvar):
            raise ValueError("state array has the wrong shape")
        eps = U[:, -1] - 0.5 * (U[:, 1:-1] * U[:, 1:-1]).sum(axis=1) / U[:, 0]
        if not ((U[:, 0] > 0.0) & (eps > 0.0)).all():
            raise AdmissibilityError("initial state is not admissible")
        Ucm = np.ascontiguousarray(U[self.cm_inv])
        lib().or_set_state(self._h, Ucm.ctypes.data)

    def get_state(self):
        Ucm = np.empty((self.n, self.nvar))
        lib().or_get_state(self._h, Ucm.ctypes.data)
        out = np.empty_like(Ucm)
        out[self.cm_inv] = Ucm
        return out

    def _check(self, st):
        if st == OR_OK:
            return
        if st == OR_TAU_UNBOUNDED:
            raise ValueError("constant field, the time step bound is unbounded")
        if st == OR_BAD_STATE:
            row = lib().or_bad_row(self._h)
            raise AdmissibilityError(f"inadmissible state at node {int(self.cm_inv[row])}")
        raise AdmissibilityError("projected state requires rho > 0 and p > 0")

    def euler_step(self, tau=None, tau_max=np.inf):
        out = ctypes.c_double()
        st = lib().or_euler_step(self._h, 0 if tau is None else 1, 0.0 if tau is None else float(tau),
                                 float(tau_max), ctypes.byref(out))
        self._check(st)
        self.tau_last = out.value
        self.n_euler_steps += 1
        return out.value

    def ssp_rk3_step(self, tau=None, tau_max=np.inf):
        out = ctypes.c_double()
        st = lib().or_ssp_rk3_step(self._h, 0 if tau is None else 1,
                                   0.0 if tau is None else float(tau), float(tau_max),
                                   ctypes.byref(out))
        self._check(st)
        self.tau_last = out.value
        self.n_euler_steps += 3
        return out.value

    def advance(self, t_final, use_rk3=True, on_step=None):
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

    _WHICH = {"d": 0, "alpha": 1, "R": 2, "bounds": 3, "l": 4, "eor": 5, "phi": 6, "U_next": 7, "P": 8}

    def fetch(self, which: str):
        """Intermediate arrays in CM row order (rows) x slot order."""
        n, L, nv = self.n, self.width, self.nvar
        shapes = {"d": (n, L), "alpha": (n,), "R": (n, nv), "bounds": (n, 3), "l": (n, L),
                  "eor": (n,), "phi": (n,), "U_next": (n, nv), "P": (n, L, nv)}
        out = np.empty(shapes[which])
        if lib().or_fetch(self._h, self._WHICH[which], out.ctypes.data) != 0:
            raise KeyError(which)
        return out


def _gas_args(gas):
    if gas is None:
        g = 7.0 / 5.0
        return (g, g - 1.0, 1.0 / (g + 1.0), (g - 1.0) / (2.0 * g), 2.0 * g / (g - 1.0))
    return (gas.gamma, gas.gm1, gas.gp1_inv, gas.gm1_over_2g, gas.two_g_over_gm1)


def eval_dij(Ui, Uj, cij, cji, gas=None):
    """riemann.d_ij_low (riemann.py:119-142) on a batch of pairs: (d, projection error flags)."""
    Ui, Uj, cij, cji = (np.ascontiguousarray(a, dtype=np.float64) for a in (Ui, Uj, cij, cji))
    n, dim = cij.shape
    out = np.empty(n)
    err = np.zeros(n, dtype=np.int32)
    lib().or_eval_dij(dim, *_gas_args(gas), n, Ui.ctypes.data, Uj.ctypes.data, cij.ctypes.data,
                      cji.ctypes.data, out.ctypes.data, err.ctypes.data)
    return out, err


def eval_limiter(U, P, bounds, newton=2, gas=None):
    """limiter.limiter_compute (limiter.py:149-193) lane by lane."""
    U, P, bounds = (np.ascontiguousarray(a, dtype=np.float64) for a in (U, P, bounds))
    n, nv = U.shape
    out = np.empty(n)
    lib().or_eval_limiter(nv - 2, *_gas_args(gas), n, U.ctypes.data, P.ctypes.data, bounds.ctypes.data,
                          int(newton), out.ctypes.data)
    return out

"""Multi-GPU: one process per GPU over NCCL, and the host-side partition plans.

The reference partitions the global Cuthill-McKee order into contiguous
ranges with one ghost layer and synchronises alpha, R, l and U between
stages plus an allreduce-min for tau (exchange.py:52-104, :160-165;
stepper.py:532-605).  Here every rank is a process bound to one GPU
(torch.distributed for the rendezvous, NCCL send/recv + allreduce inside
libef_b200.so for the data path); `partition_plan` exposes the host-only
plan so the protocol can be checked across gloo ranks on a CPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from typing import Optional

from .physics import AIR, AdmissibilityError
from .stepper import Solver, _raise, cm_permutation

__all__ = ["DistributedSolver", "ShardedSolver", "partition_plan", "partition_plan_local"]


class DistributedSolver(Solver):
    """`Solver` for one rank of a torch.distributed job (one GPU per rank).

    Every rank passes the same global matrices / state; rank r owns the r-th
    contiguous range of the CM order (exchange.py:64-70).  get_state()
    returns the full state on every rank."""

    def __init__(self, matrices, device: int = 0, **kw):
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            _raise(_lib.load().ef_nccl_unique_id(buf))
        obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=0)
        self.world = world
        self.rank = rank
        super().__init__(matrices, device=device, nccl_rank=(rank, world, obj[0]), **kw)
        from .problems import even_ranges

        given = kw.get("ranges")
        self.ranges = (np.asarray(given, dtype=np.int64) if given is not None
                       else even_ranges(self.n, world))

    def get_state(self, out=None):
        """The whole state on every rank: each rank's owned rows, gathered and
        placed by their original ids (no arithmetic on the values, so -0.0 and
        every other bit pattern survive)."""
        local = np.zeros((self.n, self.nvar))
        super().get_state(out=local)  # owned rows only
        lo, hi = int(self.ranges[self.rank]), int(self.ranges[self.rank + 1])
        res = out if out is not None else np.empty((self.n, self.nvar))
        return gather_owned_rows(local[self.cm_inv[lo:hi]], self.ranges, self.cm_inv, res)


def gather_owned_rows(mine: np.ndarray, ranges, cm_inv, out: np.ndarray) -> np.ndarray:
    """Assemble the whole state on every rank from each rank's owned rows
    (`mine`: this rank's rows of its CM range, in CM order): an all_gather of
    padded blocks, then every block placed at its rows' original ids.  Values
    are copied, never added, so every bit pattern (-0.0 included) survives."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    nvar = out.shape[1]
    width = int(max(ranges[q + 1] - ranges[q] for q in range(world)))
    buf = torch.zeros((width, nvar), dtype=torch.float64, device=dev)
    buf[:len(mine)] = torch.from_numpy(np.ascontiguousarray(mine)).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    for q in range(world):
        a, b = int(ranges[q]), int(ranges[q + 1])
        out[cm_inv[a:b]] = parts[q][:b - a].cpu().numpy()
    return out


class ShardedSolver(Solver):
    """Per-rank setup: every rank passes only its own rows
    (`problems.LocalMatrices`: owned rows + ghost layer, global ids in a node
    order chosen by the generator), so no rank holds the global matrix, a
    global permutation or an n_global-sized state.  Same kernels, halo plan
    and exchanges as `DistributedSolver`; the plans come from
    ef_create_local (include/ef_b200.h).

    parts: a single LocalMatrices (nccl=True: this process is that rank of a
    torch.distributed job, one GPU per rank), or the list of every rank's
    LocalMatrices (a same-device group, the reference's simulated ranks).
    boundary: BoundaryConditions in global ids."""

    def __init__(self, parts, c_cfl: float = 0.9, limiter_passes: int = 2, newton_steps: int = 2,
                 overlap: bool = True, boundary=None, gas=AIR, device: int = 0, stream=None,
                 nccl: bool = False):
        if not 0.0 < c_cfl <= 1.0:
            raise ValueError("c_cfl must lie in (0, 1]")
        if limiter_passes < 0:
            raise ValueError("limiter_passes must be >= 0")
        parts = [parts] if not isinstance(parts, (list, tuple)) else list(parts)
        self.parts = parts
        p0 = parts[0]
        self.gas = gas
        self.c_cfl, self.limiter_passes, self.newton_steps, self.overlap = c_cfl, limiter_passes, newton_steps, overlap
        self.bc = boundary
        self.n = int(p0.n_global)
        self.dim = int(p0.dim)
        self.nvar = self.dim + 2
        self.ranks = int(p0.nranks)
        self.ranges = np.asarray(p0.ranges, dtype=np.int64)
        self.matrices = None
        lib = _lib.load()
        keep = []

        def ptr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data

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
            stream = int(stream) or 1
        uid = None
        if nccl:
            import torch.distributed as dist

            if len(parts) != 1:
                raise ValueError("an NCCL rank passes its own LocalMatrices only")
            if dist.get_rank() != p0.rank or dist.get_world_size() != p0.nranks:
                raise ValueError("LocalMatrices rank/nranks differ from the torch.distributed job")
            buf = ctypes.create_string_buffer(128)
            if p0.rank == 0:
                _raise(lib.ef_nccl_unique_id(buf))
            obj = [bytes(buf.raw)]
            dist.broadcast_object_list(obj, src=0)
            uid = ctypes.create_string_buffer(obj[0], 128)
            keep.append(uid)
        elif len(parts) != p0.nranks or any(p.rank != r for r, p in enumerate(parts)):
            raise ValueError("a same-device group needs the LocalMatrices of ranks 0..nranks-1")
        self._handles = []
        self._group = None
        self.rank = p0.rank if nccl else 0
        self.world = p0.nranks
        self._nccl = nccl
        for lm in parts:
            loc = _lib.EfLocalMatrices(
                int(lm.n_global), int(lm.dim), int(lm.pad_width), int(lm.standard_card), int(lm.n_owned),
                len(lm.ghost_gid), ptr(lm.ghost_gid, np.int64), ptr(lm.rowptr, np.int64),
                ptr(lm.col_gid, np.int64), ptr(lm.m, np.float64), ptr(lm.c, np.float64),
                ptr(lm.m_lumped, np.float64), ptr(lm.inv_m, np.float64), ptr(lm.full_card, np.int32))
            dist_s = _lib.EfDist(int(lm.rank), int(lm.nranks), int(device), None, ptr(lm.ranges, np.int64),
                                 None if uid is None else ctypes.cast(uid, ctypes.c_void_p).value, stream)
            h = ctypes.c_void_p()
            rc = lib.ef_create_local(ctypes.byref(loc), ctypes.byref(prm), ctypes.byref(bcs),
                                     ctypes.byref(dist_s), ctypes.byref(h))
            if rc != _lib.EF_OK:
                msg = _lib.last_error()
                self.close()
                _raise(rc, msg)
            self._handles.append(h)
        if not nccl and len(self._handles) > 1:
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

    def set_state(self, U: np.ndarray):
        """NCCL rank: its owned rows (n_owned, nvar).  Group: the whole state in
        global-id order (each rank takes its range).  Collective."""
        lib = _lib.load()
        if self._nccl:
            U = np.ascontiguousarray(U, dtype=np.float64)
            if U.shape != (self.parts[0].n_owned, self.nvar):
                raise ValueError("state array has the wrong shape")
            rc = lib.ef_set_state_owned(self._h, U.ctypes.data)
        else:
            U = np.asarray(U, dtype=np.float64)
            if U.shape != (self.n, self.nvar):
                raise ValueError("state array has the wrong shape")
            if self._group is None:
                Us = [np.ascontiguousarray(U)]
                rc = lib.ef_set_state_owned(self._h, Us[0].ctypes.data)
            else:
                Us = [np.ascontiguousarray(U[self.ranges[r]:self.ranges[r + 1]]) for r in range(self.world)]
                arr = (ctypes.c_void_p * len(Us))(*[u.ctypes.data for u in Us])
                rc = lib.ef_group_set_state_owned(self._group, arr)
        if rc == _lib.EF_ERR_INADMISSIBLE:
            raise AdmissibilityError("initial state is not admissible")
        _raise(rc)

    def get_state(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """NCCL rank: its owned rows.  Group: the whole state in global-id order."""
        lib = _lib.load()
        if self._nccl or self._group is None:
            res = out if out is not None else np.empty((self.parts[0].n_owned, self.nvar))
            _raise(lib.ef_get_state_owned(self._h, res.ctypes.data))
            return res
        res = out if out is not None else np.empty((self.n, self.nvar))
        bufs = [np.empty((int(self.ranges[r + 1] - self.ranges[r]), self.nvar)) for r in range(self.world)]
        arr = (ctypes.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
        _raise(lib.ef_group_get_state_owned(self._group, arr))
        for r in range(self.world):
            res[self.ranges[r]:self.ranges[r + 1]] = bufs[r]
        return res


def partition_plan_local(lm) -> dict:
    """Host-only halo plan of one rank from its own rows (problems.LocalMatrices;
    values may be None).  Same keys as partition_plan."""
    lib = _lib.load()
    keep = []

    def ptr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a.ctypes.data

    loc = _lib.EfLocalMatrices(int(lm.n_global), int(lm.dim), int(lm.pad_width), int(lm.standard_card),
                               int(lm.n_owned), len(lm.ghost_gid), ptr(lm.ghost_gid, np.int64),
                               ptr(lm.rowptr, np.int64), ptr(lm.col_gid, np.int64), None, None, None, None, None)
    dist = _lib.EfDist(int(lm.rank), int(lm.nranks), 0, None, ptr(lm.ranges, np.int64), None, None)
    h = ctypes.c_void_p()
    _raise(lib.ef_plan_build_local(ctypes.byref(loc), ctypes.byref(dist), ctypes.byref(h)))
    return _plan_dict(lib, h, lm.nranks)


def partition_plan(matrices, rank: int, nranks: int, cm_perm=None, ranges=None) -> dict:
    """Host-only halo plan of one rank (no GPU needed).

    Returns {"n_owned", "n_local", "L", "send_rows"[q], "recv_rows"[q]}:
    rows as global CM ids in message order."""
    lib = _lib.load()
    if cm_perm is None:
        cm_perm, _ = cm_permutation(matrices)
    keep = []

    def ptr(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a.ctypes.data

    mats = _lib.EfMatrices(int(matrices.n), int(matrices.dim), ptr(matrices.indptr, np.int64),
                           ptr(matrices.indices, np.int64), None, None, None, None)
    dist = _lib.EfDist(int(rank), int(nranks), 0, ptr(cm_perm, np.int64),
                       None if ranges is None else ptr(ranges, np.int64), None, None)
    h = ctypes.c_void_p()
    _raise(lib.ef_plan_build(ctypes.byref(mats), ctypes.byref(dist), ctypes.byref(h)))
    return _plan_dict(lib, h, nranks)


def _plan_dict(lib, h, nranks) -> dict:
    try:
        sizes = np.zeros(4, dtype=np.int64)
        lib.ef_plan_sizes(h, sizes.ctypes.data)
        out = {"n_owned": int(sizes[0]), "n_local": int(sizes[1]), "L": int(sizes[2]),
               "send_rows": [], "recv_rows": []}
        for q in range(nranks):
            for recv, key in ((0, "send_rows"), (1, "recv_rows")):
                cnt = lib.ef_plan_rows(h, q, recv, None, 0)
                a = np.zeros(cnt, dtype=np.int64)
                lib.ef_plan_rows(h, q, recv, a.ctypes.data, cnt)
                out[key].append(a)
        return out
    finally:
        lib.ef_plan_destroy(h)

"""Multi-GPU: one process per GPU over NCCL, and the host-side partition plans.

The reference partitions the global Cuthill-McKee order into contiguous
ranges with one ghost layer and synchronises alpha, R, l and U between
stages plus an allreduce-min for tau (exchange.py:393-445, :160-165;
stepper.py:532-605).  Here every rank is a process bound to one GPU
(torch.distributed for the rendezvous, NCCL send/recv + allreduce inside
libef_b200.so for the data path); `partition_plan` exposes the host-only
plan so the protocol can be checked across gloo ranks on a CPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .stepper import Solver, _raise, cm_permutation

__all__ = ["DistributedSolver", "partition_plan"]


class DistributedSolver(Solver):
    """`Solver` for one rank of a torch.distributed job (one GPU per rank).

    Every rank passes the same global matrices / state; rank r owns the r-th
    contiguous range of the CM order (exchange.py:405-411).  get_state()
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
        super().__init__(matrices, device=device, nccl_rank=(rank, world, obj[0]), **kw)

    def get_state(self, out=None):
        import torch
        import torch.distributed as dist

        local = np.zeros((self.n, self.nvar))
        super().get_state(out=local)  # owned rows only
        t = torch.from_numpy(local).cuda()
        dist.all_reduce(t)  # rows are disjoint across ranks: the sum assembles them
        res = t.cpu().numpy()
        if out is not None:
            out[...] = res
            return out
        return res


def partition_plan(matrices, rank: int, nranks: int, cm_perm=None, ranges=None) -> dict:
    """Host-only halo plan of one rank (no GPU needed).

    Returns {"n_owned", "n_local", "L", "send_rows"[q], "recv_rows"[q],
    "send_slots"[q], "recv_slots"[q]}: rows as global CM ids in message
    order, slots as (row CM id, column CM id) pairs."""
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
    try:
        sizes = np.zeros(4, dtype=np.int64)
        lib.ef_plan_sizes(h, sizes.ctypes.data)
        out = {"n_owned": int(sizes[0]), "n_local": int(sizes[1]), "L": int(sizes[2]),
               "send_rows": [], "recv_rows": [], "send_slots": [], "recv_slots": []}
        for q in range(nranks):
            for recv, key in ((0, "send_rows"), (1, "recv_rows")):
                cnt = lib.ef_plan_rows(h, q, recv, None, 0)
                a = np.zeros(cnt, dtype=np.int64)
                lib.ef_plan_rows(h, q, recv, a.ctypes.data, cnt)
                out[key].append(a)
            for recv, key in ((0, "send_slots"), (1, "recv_slots")):
                cnt = lib.ef_plan_slots(h, q, recv, None, 0)
                a = np.zeros((cnt, 2), dtype=np.int64)
                lib.ef_plan_slots(h, q, recv, a.ctypes.data, cnt)
                out[key].append(a)
        return out
    finally:
        lib.ef_plan_destroy(h)

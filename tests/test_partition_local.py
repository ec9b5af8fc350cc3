"""Per-rank setup: plans built from a rank's own rows.

* the local generator's rows equal the global generator's rows bit for bit;
* the plan built from the rank's own rows (ef_plan_build_local) equals the
  plan built from the global CSR with the same global order (identity
  permutation) -- owned/local sizes and every send/receive row list;
* the 8-GPU weak-scaling point (640^3 periodic box, rank 0 of 8) builds its
  plan in bounded time and host memory without any global array."""

import os
import resource
import time

import numpy as np
import pytest

from paper_2007_00094_b200 import problems as P
from paper_2007_00094_b200.distributed import partition_plan, partition_plan_local


@pytest.mark.parametrize("n,R", [(7, 2), (9, 3), (8, 4), (6, 5)])
def test_local_plan_equals_global_plan(n, R):
    mat = P.periodic_box_matrices(n)
    ident = np.arange(mat.n, dtype=np.int64)
    for r in range(R):
        lm = P.periodic_box_local(n, r, R)
        a, b = lm.first, lm.first + lm.n_owned
        ip = mat.indptr
        assert np.array_equal(lm.col_gid[:27 * (b - a)], mat.indices[ip[a]:ip[b]])
        assert np.array_equal(lm.m[:27 * (b - a)], mat.m[ip[a]:ip[b]])
        assert np.array_equal(lm.c[:27 * (b - a)], mat.c[ip[a]:ip[b]])
        pl = partition_plan_local(lm)
        pg = partition_plan(mat, r, R, cm_perm=ident)
        assert (pl["n_owned"], pl["n_local"], pl["L"]) == (pg["n_owned"], pg["n_local"], pg["L"])
        for q in range(R):
            assert np.array_equal(pl["send_rows"][q], pg["send_rows"][q]), (r, q)
            assert np.array_equal(pl["recv_rows"][q], pg["recv_rows"][q]), (r, q)


def test_local_state_equals_global_state():
    n, R = 10, 3
    g = P.periodic_fourier_box(n)
    for r in range(R):
        lp = P.periodic_fourier_box_local(n, r, R)
        a = lp.local.first
        assert np.array_equal(lp.U0, g.U0[a:a + lp.local.n_owned])


def test_weak_scaling_640_rank0_of_8_plan_is_bounded():
    """C5 at 8 GPUs (640^3 = 262M nodes): rank 0 builds its rows' pattern and its
    halo plan from its own rows only (x-slab of 80 planes + 2 ghost planes)."""
    t0 = time.time()
    lm = P.periodic_box_local(640, 0, 8, values=False)
    plan = partition_plan_local(lm)
    dt = time.time() - t0
    rss_gb = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
    assert plan["n_owned"] == 640 ** 3 // 8
    assert plan["n_local"] - plan["n_owned"] == 2 * 640 * 640  # ghost planes x = 639 and x = 80
    assert sum(len(x) for x in plan["recv_rows"]) == 2 * 640 * 640
    assert len(plan["send_rows"][1]) == 640 * 640 and len(plan["send_rows"][7]) == 640 * 640
    print(f"640^3 rank 0 of 8: {dt:.1f} s, peak RSS {rss_gb:.1f} GB")
    assert dt < 60.0
    assert rss_gb < 64.0


@pytest.mark.parametrize("R", [1, 2, 3, 5])
def test_c4_local_rows_equal_global_rows(R):
    """C4 per rank (z-slabs of the extruded O-grid, layer-major ids): owned rows,
    ghost rows (truncated), lumped masses, cardinalities, pad width and the
    owned boundary nodes / normals equal the global generator's bit for bit."""
    ny, nz = 10, 6
    g = P.mach3_cylinder(ny, nz, shuffle=False)
    mat = g.matrices
    card = np.diff(mat.indptr)
    vals, cnt = np.unique(card, return_counts=True)
    ip = mat.indptr
    for r in range(R):
        lp = P.mach3_cylinder_local(ny, nz, r, R)
        lm = lp.local
        a, b = lm.first, lm.first + lm.n_owned
        assert lm.pad_width == card.max() and lm.standard_card == vals[np.argmax(cnt)]
        no = lm.rowptr[lm.n_owned]
        assert np.array_equal(lm.col_gid[:no], mat.indices[ip[a]:ip[b]])
        assert np.array_equal(lm.m[:no].view(np.int64), mat.m[ip[a]:ip[b]].view(np.int64))
        assert np.array_equal(lm.c[:no].view(np.int64), mat.c[ip[a]:ip[b]].view(np.int64))
        loc = np.concatenate([np.arange(a, b), lm.ghost_gid])
        assert np.array_equal(lm.m_lumped.view(np.int64), mat.m_lumped[loc].view(np.int64))
        assert np.array_equal(lm.full_card, card[loc])
        local = np.zeros(mat.n, bool)
        local[loc] = True
        for k, gid in enumerate(lm.ghost_gid):
            lo, hi = lm.rowptr[lm.n_owned + k], lm.rowptr[lm.n_owned + k + 1]
            gc = mat.indices[ip[gid]:ip[gid + 1]]
            assert np.array_equal(lm.col_gid[lo:hi], gc[local[gc]])
            assert np.array_equal(lm.m[lo:hi].view(np.int64), mat.m[ip[gid]:ip[gid + 1]][local[gc]].view(np.int64))
        bc, lbc = g.boundary, lp.boundary
        own = (bc.slip_nodes >= a) & (bc.slip_nodes < b)
        assert np.array_equal(lbc.slip_nodes, bc.slip_nodes[own])
        assert np.array_equal(lbc.slip_normals.view(np.int64), bc.slip_normals[own].view(np.int64))
        oi = (bc.inflow_nodes >= a) & (bc.inflow_nodes < b)
        if oi.any():
            assert np.array_equal(lbc.inflow_nodes, bc.inflow_nodes[oi])
        else:
            assert lbc.inflow_nodes is None
        pl = partition_plan_local(lm)
        pg = partition_plan(mat, r, R, cm_perm=np.arange(mat.n))
        assert (pl["n_owned"], pl["n_local"], pl["L"]) == (pg["n_owned"], pg["n_local"], pg["L"])
        for q in range(R):
            assert np.array_equal(pl["send_rows"][q], pg["send_rows"][q])
            assert np.array_equal(pl["recv_rows"][q], pg["recv_rows"][q])

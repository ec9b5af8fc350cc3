"""Offline inputs of the hot path: Q1 meshes, the precomputed graph matrices
and the BASELINE.json problem setups (C1-C5), vectorized.

The time step consumes only `PrecomputedMatrices` (m_ij, c_ij, m_i, 1/m_i on
a CSR stencil pattern) plus a `BoundaryConditions`, exactly the input contract
of the reference (`assembly.py:22-50`, `stepper.py:40-52`).  The reference
builds those with per-cell Python loops (`mesh.py:65-362`, `assembly.py:76-137`)
that do not scale to the 10^6-10^7-node configs, and its `assemble` rejects
uniform 3D hex meshes (beta pruning).  This module is the
vectorized replacement:

* `assemble_q1`: 2-point tensor Gauss assembly of m_ij and c_ij = ∫φ_i∇φ_j
  (same quadrature and the same exact symmetrization of m as
  `assembly.py:53-137`); beta is returned as zeros on m's pattern because the
  time step never reads it (`indicator.py:49-51`).
* mesh generators for the five BASELINE.json configs and the small reference
  problems used by the parity tests.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import os

import numpy as np
import scipy.sparse as sp

from .physics import AIR, GasConstants

__all__ = [
    "PrecomputedMatrices",
    "BoundaryConditions",
    "Mesh",
    "ProblemSetup",
    "assemble_q1",
    "assemble_q1_rows",
    "rectangle_mesh",
    "box_mesh",
    "disc_channel_mesh",
    "boundary_faces",
    "isentropic_vortex",
    "mach3_disc",
    "sod_box",
    "periodic_fourier_box",
    "periodic_box_matrices",
    "random_state",
    "make_config",
]


@dataclass
class PrecomputedMatrices:
    """Stencil-graph matrices on a canonical CSR pattern (reference `assembly.py:22-50`)."""

    n: int
    dim: int
    indptr: np.ndarray
    indices: np.ndarray
    m: np.ndarray
    c: np.ndarray
    beta: np.ndarray
    m_lumped: np.ndarray
    inv_m: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.indices)

    @property
    def card(self) -> np.ndarray:
        return np.diff(self.indptr)

    def connectivity(self) -> sp.csr_matrix:
        return sp.csr_matrix(
            (np.ones(self.nnz, dtype=np.int8), self.indices, self.indptr), shape=(self.n, self.n)
        )


@dataclass
class BoundaryConditions:
    """Strong boundary data (reference `stepper.py:40-52`); ids in original numbering."""

    inflow_nodes: Optional[np.ndarray] = None
    farfield: Optional[np.ndarray] = None
    slip_nodes: Optional[np.ndarray] = None
    slip_normals: Optional[np.ndarray] = None


@dataclass
class Mesh:
    points: np.ndarray          # (n_full, dim)
    cells: np.ndarray           # (M, 2^dim), reference corner order (mesh.py:217-231)
    dim: int
    reduced_index: Optional[np.ndarray] = None

    def __post_init__(self):
        if self.reduced_index is None:
            self.reduced_index = np.arange(len(self.points), dtype=np.int64)

    @property
    def n_nodes(self) -> int:
        return int(self.reduced_index.max()) + 1


@dataclass
class ProblemSetup:
    name: str
    matrices: PrecomputedMatrices
    U0: np.ndarray
    boundary: Optional[BoundaryConditions]
    c_cfl: float
    steps: int
    mesh: Optional[Mesh] = None
    exact: Optional[Callable] = None


_CORNERS = {
    2: np.array([(0, 0), (1, 0), (1, 1), (0, 1)], dtype=np.float64),
    3: np.array(
        [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)],
        dtype=np.float64,
    ),
}


def _shape(dim: int, xi: np.ndarray):
    corners = _CORNERS[dim]
    facs = np.where(corners > 0.5, xi[None, :], 1.0 - xi[None, :])  # (nv, dim)
    N = facs.prod(axis=1)
    dN = np.empty((len(corners), dim))
    for k in range(dim):
        other = np.delete(facs, k, axis=1).prod(axis=1)
        dN[:, k] = np.where(corners[:, k] > 0.5, 1.0, -1.0) * other
    return N, dN


def _inv_det(J: np.ndarray):
    if J.shape[-1] == 2:
        det = J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0]
        inv = np.empty_like(J)
        inv[:, 0, 0] = J[:, 1, 1]
        inv[:, 0, 1] = -J[:, 0, 1]
        inv[:, 1, 0] = -J[:, 1, 0]
        inv[:, 1, 1] = J[:, 0, 0]
        return inv / det[:, None, None], det
    det = np.linalg.det(J)
    return np.linalg.inv(J), det


def _q1_local_fn(mesh: Mesh, chunk: int):
    """Per-chunk local Q1 matrices (2-point tensor Gauss): f(cell_ids) ->
    (rows, cols, m, c) in cell order, local (a, b) row-major within a cell."""
    d = mesh.dim
    cells = mesh.cells
    red = np.asarray(mesh.reduced_index, dtype=np.int64)
    nv = cells.shape[1]
    g = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
    qpts = np.stack(np.meshgrid(*([g] * d), indexing="ij"), axis=-1).reshape(-1, d)
    w = 0.5**d
    shapes = [_shape(d, xi) for xi in qpts]

    def local(ids):  # numpy releases the GIL
        cc = cells[ids]
        X = mesh.points[cc]  # (M, nv, d)
        m_loc = np.zeros((len(cc), nv, nv))
        c_loc = np.zeros((len(cc), nv, nv, d))
        for N, dN in shapes:
            J = np.einsum("mak,al->mkl", X, dN)
            Jinv, det = _inv_det(J)
            if np.any(det <= 0.0):
                raise ValueError("degenerate cell: non-positive Jacobian determinant")
            grad = np.einsum("al,mlk->mak", dN, Jinv)
            scale = w * det
            m_loc += scale[:, None, None] * (N[:, None] * N[None, :])[None]
            c_loc += scale[:, None, None, None] * N[None, :, None, None] * grad[:, None, :, :]
        rc = red[cc]
        return (np.repeat(rc, nv, axis=1).ravel(), np.tile(rc, (1, nv)).ravel(), m_loc.ravel(),
                c_loc.reshape(-1, d))

    return local


def _local_parts(mesh: Mesh, cell_ids: np.ndarray, chunk: int):
    """Local matrices of the given cells (ascending), chunked over all host
    threads; per-cell values do not depend on the chunking."""
    from concurrent.futures import ThreadPoolExecutor

    local = _q1_local_fn(mesh, chunk)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
        return list(pool.map(lambda lo: local(cell_ids[lo:lo + chunk]), range(0, len(cell_ids), chunk)))


def assemble_q1_rows(mesh: Mesh, slabs: int, chunk: int = 1 << 15) -> PrecomputedMatrices:
    """`assemble_q1` one range of rows at a time (memory ~1/slabs of it): the
    rows of a range take the same cell contributions in the same order, so every
    value is bit-identical.  For meshes whose cells never repeat a node (m is
    then exactly symmetric, so the symmetrisation is the identity); used for the
    8.4M-node C3 box."""
    d = mesh.dim
    n = mesh.n_nodes
    red = np.asarray(mesh.reduced_index, dtype=np.int64)
    rc_all = red[mesh.cells]
    if np.any(np.sort(rc_all, axis=1)[:, 1:] == np.sort(rc_all, axis=1)[:, :-1]):
        raise ValueError("assemble_q1_rows needs cells with distinct nodes")
    bounds = np.linspace(0, n, slabs + 1).astype(np.int64)
    counts = np.zeros(n, dtype=np.int64)
    idx_parts, m_parts, c_parts = [], [], []
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        if r1 <= r0:
            continue
        cell_ids = np.flatnonzero(((rc_all >= r0) & (rc_all < r1)).any(axis=1))
        parts = _local_parts(mesh, cell_ids, chunk)
        rows = np.concatenate([q[0] for q in parts])
        keep = (rows >= r0) & (rows < r1)
        rows = rows[keep]
        cols = np.concatenate([q[1] for q in parts])[keep]
        mv = np.concatenate([q[2] for q in parts])[keep]
        cv = np.concatenate([q[3] for q in parts])[keep]
        del parts, keep
        key = rows * n + cols
        order = np.argsort(key, kind="stable")
        key = key[order]
        first = np.ones(len(key), dtype=bool)
        first[1:] = key[1:] != key[:-1]
        seg = np.flatnonzero(first)
        m_parts.append(np.add.reduceat(mv[order], seg))
        c_parts.append(np.add.reduceat(cv[order], seg, axis=0))
        ukey = key[seg]
        idx_parts.append((ukey % n).astype(np.int64))
        counts[r0:r1] = np.bincount(ukey // n - r0, minlength=r1 - r0)
        del rows, cols, mv, cv, key, order, first, seg, ukey
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    indices = np.concatenate(idx_parts)
    m_data = np.concatenate(m_parts)
    del idx_parts, m_parts
    c_data = np.concatenate(c_parts)
    del c_parts
    m_sym = 0.5 * (m_data + m_data)  # = m exactly: the local mass matrices are symmetric
    m_lumped = np.add.reduceat(m_sym, indptr[:-1])
    if np.any(m_lumped <= 0.0):
        raise ValueError("non-positive lumped mass entry")
    return PrecomputedMatrices(
        n=n, dim=d, indptr=indptr, indices=indices, m=m_sym, c=c_data,
        beta=np.zeros(0), m_lumped=m_lumped, inv_m=1.0 / m_lumped,
    )


def assemble_q1(mesh: Mesh, chunk: int = 1 << 15) -> PrecomputedMatrices:
    """Assemble m_ij, c_ij and the lumped mass on the Q1 stencil graph."""
    n = mesh.n_nodes
    d = mesh.dim
    parts = _local_parts(mesh, np.arange(len(mesh.cells)), chunk)
    rows_all = [q[0] for q in parts]
    cols_all = [q[1] for q in parts]
    mv_all = [q[2] for q in parts]
    cv_all = [q[3] for q in parts]
    del parts
    rows = np.concatenate(rows_all)
    cols = np.concatenate(cols_all)
    mv = np.concatenate(mv_all)
    cv = np.concatenate(cv_all)
    del rows_all, cols_all, mv_all, cv_all

    # canonical pattern: sort by (row, col), sum duplicates in a fixed order
    key = rows * n + cols
    order = np.argsort(key, kind="stable")
    key = key[order]
    first = np.ones(len(key), dtype=bool)
    first[1:] = key[1:] != key[:-1]
    seg = np.flatnonzero(first)
    m_data = np.add.reduceat(mv[order], seg)
    c_data = np.add.reduceat(cv[order], seg, axis=0)
    ukey = key[seg]
    r_u = ukey // n
    indices = (ukey % n).astype(np.int64)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, r_u + 1, 1)
    indptr = np.cumsum(indptr)
    # exact symmetry of m (as assembly.py:113): 0.5 * (m + m^T) on the shared pattern
    mat = sp.csr_matrix((m_data, indices, indptr), shape=(n, n))
    mt = mat.T.tocsr()
    mt.sort_indices()
    if not (np.array_equal(mt.indptr, indptr) and np.array_equal(mt.indices, indices)):
        raise AssertionError("stencil pattern is not structurally symmetric")
    m_sym = 0.5 * (m_data + mt.data)
    m_lumped = np.add.reduceat(m_sym, indptr[:-1])
    if np.any(m_lumped <= 0.0):
        raise ValueError("non-positive lumped mass entry")
    return PrecomputedMatrices(
        n=n, dim=d, indptr=indptr, indices=indices, m=m_sym, c=c_data,
        beta=np.zeros_like(m_sym), m_lumped=m_lumped, inv_m=1.0 / m_lumped,
    )


# --------------------------------------------------------------------------- meshes

def rectangle_mesh(nx, ny, x_range=(0.0, 1.0), y_range=(0.0, 1.0), periodic=(False, False)) -> Mesh:
    xs = np.linspace(*x_range, nx + 1)
    ys = np.linspace(*y_range, ny + 1)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    pts = np.column_stack([X.ravel(), Y.ravel()])
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    i, j = i.ravel(), j.ravel()
    nid = lambda a, b: a * (ny + 1) + b  # noqa: E731
    cells = np.stack([nid(i, j), nid(i + 1, j), nid(i + 1, j + 1), nid(i, j + 1)], axis=1)
    ri = np.arange(nx + 1)
    rj = np.arange(ny + 1)
    if periodic[0]:
        ri[nx] = 0
    if periodic[1]:
        rj[ny] = 0
    rep = (ri[:, None] * (ny + 1) + rj[None, :]).ravel()
    _, reduced = np.unique(rep, return_inverse=True)
    return Mesh(points=pts, cells=cells.astype(np.int64), dim=2, reduced_index=reduced.astype(np.int64))


def box_mesh(nx, ny, nz, x_range=(0.0, 1.0), y_range=(0.0, 1.0), z_range=(0.0, 1.0),
             periodic=(False, False, False), jitter=0.0, seed=0) -> Mesh:
    """Tensor hex mesh with nx*ny*nz cells; interior nodes optionally jittered
    i.i.d. U(-jitter*h, jitter*h) per axis (BASELINE C3)."""
    xs = np.linspace(*x_range, nx + 1)
    ys = np.linspace(*y_range, ny + 1)
    zs = np.linspace(*z_range, nz + 1)
    X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
    pts = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])
    if jitter > 0.0:
        rng = np.random.default_rng(seed)
        h = np.array([(x_range[1] - x_range[0]) / nx, (y_range[1] - y_range[0]) / ny,
                      (z_range[1] - z_range[0]) / nz])
        I, J, K = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
        interior = ((I > 0) & (I < nx) & (J > 0) & (J < ny) & (K > 0) & (K < nz)).ravel()
        pts[interior] += rng.uniform(-jitter, jitter, (int(interior.sum()), 3)) * h
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    nid = lambda a, b, c: (a * (ny + 1) + b) * (nz + 1) + c  # noqa: E731
    cells = np.stack([
        nid(i, j, k), nid(i + 1, j, k), nid(i + 1, j + 1, k), nid(i, j + 1, k),
        nid(i, j, k + 1), nid(i + 1, j, k + 1), nid(i + 1, j + 1, k + 1), nid(i, j + 1, k + 1),
    ], axis=1)
    ri, rj, rk = np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1)
    if periodic[0]:
        ri[nx] = 0
    if periodic[1]:
        rj[ny] = 0
    if periodic[2]:
        rk[nz] = 0
    rep = ((ri[:, None, None] * (ny + 1) + rj[None, :, None]) * (nz + 1) + rk[None, None, :]).ravel()
    if any(periodic):
        _, reduced = np.unique(rep, return_inverse=True)
        reduced = reduced.astype(np.int64)
    else:
        reduced = None
    return Mesh(points=pts, cells=cells.astype(np.int64), dim=3, reduced_index=reduced)


def disc_channel_mesh(ny: int, center=(0.6, 0.5), radius=0.1, half_box=0.2,
                      x_len=4.0, y_len=1.0, grading=1.04) -> Mesh:
    """Channel [0,x_len]x[0,y_len] minus a disc: a uniform Cartesian far field of
    spacing h = y_len/ny whose square block [c-a, c+a]^2 is replaced by a graded
    quad O-grid from the square perimeter to the circle (BASELINE C2 geometry)."""
    h = y_len / ny
    nx = int(round(x_len / h))
    cx, cy = center
    na = int(round(half_box / h))
    i0, i1 = int(round((cx - half_box) / h)), int(round((cx + half_box) / h))
    j0, j1 = int(round((cy - half_box) / h)), int(round((cy + half_box) / h))
    if i1 - i0 != 2 * na or j1 - j0 != 2 * na:
        raise ValueError("disc box must align with the grid; choose ny accordingly")
    xs = np.linspace(0.0, x_len, nx + 1)
    ys = np.linspace(0.0, y_len, ny + 1)
    I, J = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), indexing="ij")
    inside = (I > i0) & (I < i1) & (J > j0) & (J < j1)
    keep = ~inside.ravel()
    gid = np.full((nx + 1) * (ny + 1), -1, dtype=np.int64)
    gid[keep] = np.arange(int(keep.sum()))
    pts = np.column_stack([xs[I.ravel()], ys[J.ravel()]])[keep]
    ci, cj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    ci, cj = ci.ravel(), cj.ravel()
    cell_in = (ci >= i0) & (ci < i1) & (cj >= j0) & (cj < j1)
    ci, cj = ci[~cell_in], cj[~cell_in]
    nid = lambda a, b: gid[a * (ny + 1) + b]  # noqa: E731
    cells = [np.stack([nid(ci, cj), nid(ci + 1, cj), nid(ci + 1, cj + 1), nid(ci, cj + 1)], axis=1)]

    # square perimeter, counterclockwise from (i0, j0)
    side = 2 * na
    pi = np.concatenate([np.arange(i0, i1), np.full(side, i1), np.arange(i1, i0, -1), np.full(side, i0)])
    pj = np.concatenate([np.full(side, j0), np.arange(j0, j1), np.full(side, j1), np.arange(j1, j0, -1)])
    ring0 = nid(pi, pj)
    S = np.column_stack([xs[pi], ys[pj]])
    v = S - np.array(center)
    rS = np.linalg.norm(v, axis=1)
    C = np.array(center) + radius * v / rS[:, None]
    # graded radial layers: tangential spacing at the disc -> h at the box
    P = len(ring0)
    dr_min = 2.0 * np.pi * radius / P
    nlay = max(2, int(np.ceil((half_box - radius) / (0.5 * (dr_min + h)))))
    q = (h / dr_min) ** (1.0 / nlay)
    s = (q ** np.arange(0, nlay + 1) - 1.0) / (q**nlay - 1.0)  # s[0]=0 disc, s[nlay]=1 box
    rings = [ring0]
    base = len(pts)
    new_pts = []
    for k in range(nlay - 1, 0, -1):  # interior rings from the box inward (s decreasing)
        new_pts.append(C + s[k] * (S - C))
        rings.append(base + np.arange(P))
        base += P
    new_pts.append(C)
    rings.append(base + np.arange(P))
    pts = np.concatenate([pts] + new_pts)
    for a, b in zip(rings[:-1], rings[1:]):
        an = np.roll(a, -1)
        bn = np.roll(b, -1)
        cells.append(np.stack([a, an, bn, b], axis=1))
    cells = np.concatenate(cells).astype(np.int64)
    # orient all cells counterclockwise (positive Jacobian)
    X = pts[cells]
    area2 = ((X[:, 1, 0] - X[:, 0, 0]) * (X[:, 3, 1] - X[:, 0, 1])
             - (X[:, 1, 1] - X[:, 0, 1]) * (X[:, 3, 0] - X[:, 0, 0]))
    flip = area2 < 0
    cells[flip] = cells[flip][:, [0, 3, 2, 1]]
    return Mesh(points=pts, cells=cells, dim=2)


_LOCAL_FACES = {
    2: np.array([(0, 1), (1, 2), (2, 3), (3, 0)]),
    3: np.array([(0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7)]),
}


def boundary_faces(mesh: Mesh):
    """Vectorized `mesh.boundary_faces` (reference mesh.py:318-362): faces that
    belong to exactly one cell, their outward unit normals and measures."""
    d = mesh.dim
    lf = _LOCAL_FACES[d]
    faces = mesh.cells[:, lf].reshape(-1, lf.shape[1])
    owner = np.repeat(np.arange(len(mesh.cells)), len(lf))
    red = mesh.reduced_index[faces]
    key = np.sort(red, axis=1)
    _, inv, counts = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    single = counts[inv.ravel()] == 1
    faces = faces[single]
    owner = owner[single]
    P = mesh.points[faces]
    if d == 2:
        t = P[:, 1] - P[:, 0]
        normal = np.column_stack([t[:, 1], -t[:, 0]])
        measure = np.linalg.norm(t, axis=1)
    else:
        normal = 0.5 * np.cross(P[:, 2] - P[:, 0], P[:, 3] - P[:, 1])
        measure = np.linalg.norm(normal, axis=1)
    nn = np.linalg.norm(normal, axis=1)
    normal = normal / np.where(nn > 0, nn, 1.0)[:, None]
    outward = P.mean(axis=1) - mesh.points[mesh.cells[owner]].mean(axis=1)
    flip = (normal * outward).sum(axis=1) < 0
    normal[flip] *= -1.0
    return faces, normal, measure


def _conserved(rho, vel, p, gas: GasConstants):
    U = np.empty((len(rho), vel.shape[1] + 2))
    U[:, 0] = rho
    U[:, 1:-1] = rho[:, None] * vel
    U[:, -1] = p / gas.gm1 + 0.5 * rho * (vel * vel).sum(axis=1)
    return U


def _slip_inflow_bc(mesh: Mesh, inflow_mask_fn, outflow_mask_fn, farfield):
    """Classify boundary nodes as in `problems.mach3_channel` (problems.py:49-80)."""
    faces, normals, measures = boundary_faces(mesh)
    red = mesh.reduced_index
    n = mesh.n_nodes
    fx = mesh.points[faces]  # (nf, k, d)
    is_in = inflow_mask_fn(fx).all(axis=1) if inflow_mask_fn else np.zeros(len(faces), bool)
    is_out = outflow_mask_fn(fx).all(axis=1) if outflow_mask_fn else np.zeros(len(faces), bool)
    is_out &= ~is_in
    slip_f = ~(is_in | is_out)
    inflow = np.zeros(n, dtype=bool)
    inflow[red[faces[is_in]].ravel()] = True
    slip = np.zeros(n, dtype=bool)
    slip[red[faces[slip_f]].ravel()] = True
    acc = np.zeros((n, mesh.dim))
    contrib = (measures[slip_f, None] * normals[slip_f])
    for k in range(faces.shape[1]):
        np.add.at(acc, red[faces[slip_f, k]], contrib)
    slip &= ~inflow
    slip_nodes = np.flatnonzero(slip)
    nrm = acc[slip_nodes]
    ln = np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm = nrm / np.where(ln > 0.0, ln, 1.0)
    return BoundaryConditions(
        inflow_nodes=np.flatnonzero(inflow) if inflow.any() else None,
        farfield=np.asarray(farfield, dtype=np.float64) if farfield is not None else None,
        slip_nodes=slip_nodes if len(slip_nodes) else None,
        slip_normals=nrm if len(slip_nodes) else None,
    )


# --------------------------------------------------------------------------- problems

def isentropic_vortex(n: int = 128, beta: float = 5.0, gas: GasConstants = AIR,
                      steps: int = 100) -> ProblemSetup:
    """BASELINE C1: [-5,5]^2, (n+1)^2 nodes, vortex on (rho, u, p) = (1, (1,1), 1);
    Dirichlet far field = background state on every boundary node."""
    mesh = rectangle_mesh(n, n, (-5.0, 5.0), (-5.0, 5.0))
    mat = assemble_q1(mesh)
    x, y = mesh.points[:, 0], mesh.points[:, 1]
    r2 = x * x + y * y
    g = gas.gamma
    e = np.exp(0.5 * (1.0 - r2))
    du = -beta / (2.0 * np.pi) * e * y
    dv = beta / (2.0 * np.pi) * e * x
    T = 1.0 - (g - 1.0) * beta**2 / (8.0 * g * np.pi**2) * np.exp(1.0 - r2)
    rho = T ** (1.0 / (g - 1.0))
    p = rho**g
    U0 = _conserved(rho, np.column_stack([1.0 + du, 1.0 + dv]), p, gas)
    ff = _conserved(np.array([1.0]), np.array([[1.0, 1.0]]), np.array([1.0]), gas)[0]
    on_bnd = (np.abs(np.abs(x) - 5.0) < 1e-12) | (np.abs(np.abs(y) - 5.0) < 1e-12)
    bc = BoundaryConditions(inflow_nodes=np.flatnonzero(on_bnd), farfield=ff)
    return ProblemSetup("c1-vortex", mat, U0, bc, c_cfl=0.5, steps=steps, mesh=mesh)


def mach3_disc(ny: int = 550, seed: int = 2007, gas: GasConstants = AIR,
               steps: int = 200, shuffle: bool = True) -> ProblemSetup:
    """BASELINE C2: Mach 3 past a disc r=0.1 at (0.6,0.5) in [0,4]x[0,1]; ny=550
    gives ~1.24M nodes.  Node ids are shuffled with a seeded permutation (the
    solver applies RCM itself).  Inflow x=0, do-nothing x=4, slip elsewhere."""
    mesh = disc_channel_mesh(ny)
    if shuffle:
        perm = np.random.default_rng(seed).permutation(len(mesh.points))  # old -> new
        pts = np.empty_like(mesh.points)
        pts[perm] = mesh.points
        mesh = Mesh(points=pts, cells=perm[mesh.cells], dim=2)
    mat = assemble_q1(mesh)
    ff = _conserved(np.array([1.4]), np.array([[3.0, 0.0]]), np.array([1.0]), gas)[0]
    bc = _slip_inflow_bc(mesh, lambda X: X[..., 0] < 1e-9, lambda X: X[..., 0] > 4.0 - 1e-9, ff)
    U0 = np.tile(ff, (mat.n, 1))
    return ProblemSetup("c2-mach3-disc", mat, U0, bc, c_cfl=0.9, steps=steps, mesh=mesh)


def sod_box(nx: int = 511, ny: int = 127, nz: int = 127, jitter: float = 0.2, seed: int = 2007,
            gas: GasConstants = AIR, steps: int = 100) -> ProblemSetup:
    """BASELINE C3: [0,1]x[0,.25]^2 hex box, (nx+1)(ny+1)(nz+1) nodes, interior
    jitter ±0.2h, Sod states split at x=0.5, slip walls."""
    mesh = box_mesh(nx, ny, nz, (0.0, 1.0), (0.0, 0.25), (0.0, 0.25), jitter=jitter, seed=seed)
    cells = len(mesh.cells)  # full C3: row ranges of ~0.5M cells keep host memory ~10x lower
    mat = assemble_q1(mesh) if cells <= (1 << 21) else assemble_q1_rows(mesh, slabs=-(-cells // (1 << 19)))
    left = mesh.points[:, 0] < 0.5
    rho = np.where(left, 1.0, 0.125)
    p = np.where(left, 1.0, 0.1)
    U0 = _conserved(rho, np.zeros((len(rho), 3)), p, gas)
    bc = _slip_inflow_bc(mesh, None, None, None)
    return ProblemSetup("c3-sod-box", mat, U0, bc, c_cfl=0.9, steps=steps, mesh=mesh)


def extrude(mesh2d: Mesh, nz: int, z_range=(0.0, 1.0)) -> Mesh:
    """Hex mesh from a 2D quad mesh extruded over nz uniform layers in z; the
    quad (a, b, c, d) of layer k gives the hex (a, b, c, d) at z_k then at
    z_{k+1}, the reference corner order of a counterclockwise quad."""
    if mesh2d.dim != 2:
        raise ValueError("extrude needs a 2D mesh")
    n2 = len(mesh2d.points)
    zs = np.linspace(z_range[0], z_range[1], nz + 1)
    pts = np.empty(((nz + 1) * n2, 3))
    pts[:, :2] = np.tile(mesh2d.points, (nz + 1, 1))
    pts[:, 2] = np.repeat(zs, n2)
    q = mesh2d.cells
    k = np.arange(nz, dtype=np.int64)[:, None, None] * n2
    cells = np.concatenate([q[None] + k, q[None] + k + n2], axis=2).reshape(-1, 8)
    return Mesh(points=pts, cells=cells.astype(np.int64), dim=3)


def mach3_cylinder(ny: int = 255, nz: int = 255, seed: int = 2007, gas: GasConstants = AIR,
                   steps: int = 50, shuffle: bool = True) -> ProblemSetup:
    """BASELINE C4: Mach 3 past a cylinder r=0.1 along z at (0.6, 0.5) in
    [0,4]x[0,1]x[0,1]: the C2 O-grid (`disc_channel_mesh(ny)`) extruded over nz
    layers.  ny = nz = 255 gives ~67M nodes (8 GPUs); smaller ny/nz give
    single-GPU and oracle-sized instances.  Inflow x=0 (rho=1.4, u=(3,0,0),
    p=1), do-nothing x=4, slip on the cylinder and the four side walls."""
    mesh = extrude(disc_channel_mesh(ny), nz)
    if shuffle:
        perm = np.random.default_rng(seed).permutation(len(mesh.points))  # old -> new
        pts = np.empty_like(mesh.points)
        pts[perm] = mesh.points
        mesh = Mesh(points=pts, cells=perm[mesh.cells], dim=3)
    mat = assemble_q1(mesh)
    ff = _conserved(np.array([1.4]), np.array([[3.0, 0.0, 0.0]]), np.array([1.0]), gas)[0]
    bc = _slip_inflow_bc(mesh, lambda X: X[..., 0] < 1e-9, lambda X: X[..., 0] > 4.0 - 1e-9, ff)
    U0 = np.tile(ff, (mat.n, 1))
    return ProblemSetup("c4-mach3-cylinder", mat, U0, bc, c_cfl=0.9, steps=steps, mesh=mesh)


def _periodic_stencil(n: int):
    """The translation-invariant 27-point Q1 stencil of the periodic n^3 box:
    offsets, m per offset (symmetrised exactly), c per offset, lumped mass."""
    if n < 3:
        raise ValueError("periodic box needs n >= 3")
    h = 1.0 / n
    cell = Mesh(points=_CORNERS[3] * h, cells=np.arange(8)[None, :], dim=3)
    loc = assemble_q1(cell)  # one cell: a dense 8x8 pattern
    m_loc = np.zeros((8, 8))
    c_loc = np.zeros((8, 8, 3))
    for a in range(8):
        for q in range(loc.indptr[a], loc.indptr[a + 1]):
            m_loc[a, loc.indices[q]] = loc.m[q]
            c_loc[a, loc.indices[q]] = loc.c[q]
    corners = _CORNERS[3].astype(np.int64)
    offs = np.array([(x, y, z) for x in (-1, 0, 1) for y in (-1, 0, 1) for z in (-1, 0, 1)])
    m_off = np.zeros(27)
    c_off = np.zeros((27, 3))
    for k, o in enumerate(offs):
        for a in range(8):  # node 0 is local vertex a of the cell with origin -corners[a]
            b = np.flatnonzero((corners == corners[a] + o).all(axis=1))
            if len(b):
                m_off[k] += m_loc[a, b[0]]
                c_off[k] += c_loc[a, b[0]]
    mirror = np.array([np.flatnonzero((offs == -o).all(axis=1))[0] for o in offs])
    m_sym = 0.5 * (m_off + m_off[mirror])
    m_i = m_sym[0]
    for k in range(1, 27):
        m_i = m_i + m_sym[k]
    return offs, m_sym, c_off, m_i


def _periodic_rows(n: int, ids: np.ndarray, offs, m_sym, c_off, values: bool = True):
    """Stencils of the rows `ids` (node id = (ix n + iy) n + iz) of the periodic
    box: columns ascending, with the matching m and c.  Away from the periodic
    seams every row's columns are i + flat(o), already sorted by the offsets'
    flat order; only the seam rows need a per-row sort."""
    ids = np.asarray(ids, dtype=np.int64)
    flat = (offs[:, 0] * n + offs[:, 1]) * n + offs[:, 2]
    base_order = np.argsort(flat, kind="stable")
    cols = ids[:, None] + flat[base_order][None, :]
    m = c = None
    if values:
        m = np.broadcast_to(m_sym[base_order], (len(ids), 27)).copy()
        c = np.broadcast_to(c_off[base_order], (len(ids), 27, 3)).copy()
    ix, iy, iz = np.unravel_index(ids, (n, n, n))
    seam = np.flatnonzero((ix == 0) | (ix == n - 1) | (iy == 0) | (iy == n - 1) | (iz == 0) | (iz == n - 1))
    sx, sy, sz = ix[seam], iy[seam], iz[seam]
    del ix, iy, iz
    sc = np.empty((len(seam), 27), dtype=np.int64)
    for k, o in enumerate(offs):
        sc[:, k] = (((sx + o[0]) % n) * n + (sy + o[1]) % n) * n + (sz + o[2]) % n
    order = np.argsort(sc, axis=1, kind="stable")
    cols[seam] = np.take_along_axis(sc, order, axis=1)
    if values:
        m[seam] = m_sym[order]
        c[seam] = c_off[order]
    return cols, m, c


def periodic_box_matrices(n: int) -> PrecomputedMatrices:
    """Q1 matrices of the uniform periodic n^3 hex mesh of the unit cube, built
    from its translation invariance (every node has the same 27-point stencil
    values) instead of a per-cell assembly -- O(n^3) memory and time, so the
    262M-node C5 instance is feasible.  The values are those of `assemble_q1`
    (same quadrature; the per-offset sums are taken over the 8 cells around a
    node in a fixed order and m is symmetrised exactly)."""
    offs, m_sym, c_off, m_i = _periodic_stencil(n)
    N = n ** 3
    cols, m, c = _periodic_rows(n, np.arange(N, dtype=np.int64), offs, m_sym, c_off)
    m = m.ravel()
    c = c.reshape(-1, 3)
    m_lumped = np.full(N, m_i)
    return PrecomputedMatrices(n=N, dim=3, indptr=np.arange(0, 27 * N + 1, 27, dtype=np.int64),
                               indices=cols.ravel(), m=m, c=c, beta=np.zeros(0), m_lumped=m_lumped,
                               inv_m=1.0 / m_lumped)


@dataclass
class LocalMatrices:
    """One rank's rows of a PrecomputedMatrices (per-rank setup, ef_local_matrices in
    include/ef_b200.h): owned rows [ranges[rank], ranges[rank+1]) with full stencils,
    then the ghost rows (ascending global id) truncated to local columns; global
    column ids ascending per row."""
    n_global: int
    dim: int
    pad_width: int
    standard_card: int
    rank: int
    nranks: int
    ranges: np.ndarray
    ghost_gid: np.ndarray
    rowptr: np.ndarray
    col_gid: np.ndarray
    m: Optional[np.ndarray]
    c: Optional[np.ndarray]
    m_lumped: np.ndarray
    inv_m: np.ndarray
    full_card: np.ndarray

    @property
    def n_owned(self) -> int:
        return int(self.ranges[self.rank + 1] - self.ranges[self.rank])

    @property
    def first(self) -> int:
        return int(self.ranges[self.rank])


def even_ranges(n: int, nranks: int) -> np.ndarray:
    """exchange.partition's split (exchange.py:64-70)."""
    base, extra = divmod(n, nranks)
    sizes = [base + (1 if r < extra else 0) for r in range(nranks)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def periodic_box_local(n: int, rank: int, nranks: int, values: bool = True) -> LocalMatrices:
    """Rank `rank`'s rows of periodic_box_matrices(n) in the box's lexicographic
    node order (x slowest: contiguous ranges are x-slabs), without building the
    global matrix: O(n^3 / nranks) host memory and time.  Each row equals the
    matching row of periodic_box_matrices(n) bit for bit (same stencil routine)."""
    offs, m_sym, c_off, m_i = _periodic_stencil(n)
    N = n ** 3
    ranges = even_ranges(N, nranks)
    a, b = int(ranges[rank]), int(ranges[rank + 1])
    own_cols, own_m, own_c = _periodic_rows(n, np.arange(a, b, dtype=np.int64), offs, m_sym, c_off, values)
    off = own_cols[(own_cols < a) | (own_cols >= b)]
    ghosts = np.unique(off)
    del off
    g_cols, g_m, g_c = _periodic_rows(n, ghosts, offs, m_sym, c_off, values)
    keep = ((g_cols >= a) & (g_cols < b)) | np.isin(g_cols, ghosts)
    g_card = keep.sum(axis=1)
    n_own = b - a
    rowptr = np.empty(n_own + len(ghosts) + 1, dtype=np.int64)
    rowptr[0] = 0
    rowptr[1:n_own + 1] = 27 * np.arange(1, n_own + 1, dtype=np.int64)
    rowptr[n_own + 1:] = 27 * n_own + np.cumsum(g_card)
    col_gid = np.concatenate([own_cols.ravel(), g_cols[keep]])
    del own_cols
    m = c = None
    if values:
        m = np.concatenate([own_m.ravel(), g_m[keep]])
        c = np.concatenate([own_c.reshape(-1, 3), g_c[keep]])
    n_loc = n_own + len(ghosts)
    m_lumped = np.full(n_loc, m_i)
    return LocalMatrices(n_global=N, dim=3, pad_width=27, standard_card=27, rank=rank, nranks=nranks,
                         ranges=ranges, ghost_gid=ghosts.astype(np.int64), rowptr=rowptr, col_gid=col_gid,
                         m=m, c=c, m_lumped=m_lumped, inv_m=1.0 / m_lumped,
                         full_card=np.full(n_loc, 27, dtype=np.int32))


def _fourier_state(n: int, ids: np.ndarray, seed: int, gas: GasConstants, modes: int = 8) -> np.ndarray:
    """The C5 initial state at the nodes `ids` (elementwise in a fixed order:
    independent of which rows are evaluated together)."""
    ix, iy, iz = np.unravel_index(np.asarray(ids, dtype=np.int64), (n, n, n))
    rep = np.column_stack([ix, iy, iz]) / float(n)
    del ix, iy, iz
    rng = np.random.default_rng(seed)
    fields = []
    chunk = 1 << 20  # row chunks evaluated on all host threads (numpy releases the GIL)
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
        for _ in range(5):
            k = rng.integers(-2, 3, (modes, 3))
            while np.any(np.all(k == 0, axis=1)):
                bad = np.all(k == 0, axis=1)
                k[bad] = rng.integers(-2, 3, (int(bad.sum()), 3))
            a = rng.uniform(-1.0, 1.0, modes)
            ph = rng.uniform(0.0, 2.0 * np.pi, modes)
            gsum = np.empty(len(rep))

            def part(lo, k=k, a=a, ph=ph, gsum=gsum):
                r = rep[lo:lo + chunk]
                acc = np.zeros(len(r))
                for q in range(modes):
                    kx = (r[:, 0] * k[q, 0] + r[:, 1] * k[q, 1]) + r[:, 2] * k[q, 2]
                    acc += a[q] * np.sin(2.0 * np.pi * kx + ph[q])
                gsum[lo:lo + chunk] = acc

            list(pool.map(part, range(0, len(rep), chunk)))
            fields.append(gsum / np.abs(a).sum())
    rho = 1.0 + 0.5 * fields[0]
    p = 1.0 + 0.5 * fields[1]
    vel = np.column_stack(fields[2:5]) / np.sqrt(3.0)
    return _conserved(rho, vel, p, gas)


@dataclass
class LocalProblem:
    """One rank's share of a problem (per-rank setup): its rows and its owned states."""
    name: str
    local: LocalMatrices
    U0: np.ndarray          # (n_owned, nvar): owned rows, global-id order
    c_cfl: float
    steps: int
    boundary: Optional[BoundaryConditions] = None  # global ids, owned rows only


def periodic_fourier_box_local(n: int, rank: int, nranks: int, seed: int = 2007, gas: GasConstants = AIR,
                               steps: int = 50) -> LocalProblem:
    """Rank `rank`'s share of periodic_fourier_box(n) (C5 weak scaling: 320^3 per
    GPU, n = round(320 N^(1/3))).  Rows and states equal those of the global
    generator for the same global ids."""
    lm = periodic_box_local(n, rank, nranks)
    U0 = _fourier_state(n, np.arange(lm.first, lm.first + lm.n_owned, dtype=np.int64), seed, gas)
    return LocalProblem("c5-periodic-box", lm, U0, c_cfl=0.9, steps=steps)


def periodic_fourier_box(n: int = 320, seed: int = 2007, gas: GasConstants = AIR,
                         steps: int = 50, modes: int = 8) -> ProblemSetup:
    """BASELINE C5: periodic n^3 hex mesh; rho, p in [0.5,1.5], |u| <= 1 from a
    sum of `modes` random low-frequency Fourier modes per field."""
    mat = periodic_box_matrices(n)
    U0 = _fourier_state(n, np.arange(mat.n, dtype=np.int64), seed, gas, modes)
    return ProblemSetup("c5-periodic-box", mat, U0, None, c_cfl=0.9, steps=steps, mesh=None)


def _q1_cardinality(mesh: Mesh) -> np.ndarray:
    """Stencil cardinality of every node of a Q1 mesh (the nodes sharing a cell)."""
    k = mesh.cells.shape[1]
    rows = np.repeat(mesh.cells, k, axis=1).ravel()
    cols = np.tile(mesh.cells, (1, k)).ravel()
    n = len(mesh.points)
    conn = sp.csr_matrix((np.ones(len(rows), dtype=np.int8), (rows, cols)), shape=(n, n))
    conn.sum_duplicates()
    return np.diff(conn.indptr)


def mach3_cylinder_local(ny: int = 255, nz: int = 255, rank: int = 0, nranks: int = 1,
                         gas: GasConstants = AIR, steps: int = 50) -> LocalProblem:
    """Rank `rank`'s share of mach3_cylinder(ny, nz, shuffle=False) (BASELINE C4),
    built without the global mesh: node ids are layer-major (extrude order), so
    a contiguous range of them is a z-slab.  The rank assembles only the cell
    layers around its slab (its owned and ghost rows need every cell they touch:
    node layers la-2 .. lb+2 for owned layers la .. lb), with the global node
    ids and cell order restricted, so every row value, lumped mass and boundary
    normal of its owned rows (and the row values of its ghost rows) equals the
    global generator's bit for bit (tests/test_partition_local.py).  Host memory
    ~1/nranks of the global assembly: the 67M-node C4 at 8 GPUs is 8.4M rows a
    rank.  Boundary lists are in global ids, owned rows only."""
    m2 = disc_channel_mesh(ny)
    n2 = len(m2.points)
    zs = np.linspace(0.0, 1.0, nz + 1)  # extrude's z values
    N = (nz + 1) * n2
    ranges = even_ranges(N, nranks)
    a, b = int(ranges[rank]), int(ranges[rank + 1])
    la, lb = a // n2, (b - 1) // n2
    c0, c1 = max(la - 2, 0), min(lb + 1, nz - 1)  # cell layers
    n0, n1 = c0, c1 + 1                           # node layers of the sub-mesh
    pts = np.empty(((n1 - n0 + 1) * n2, 3))
    pts[:, :2] = np.tile(m2.points, (n1 - n0 + 1, 1))
    pts[:, 2] = np.repeat(zs[n0:n1 + 1], n2)
    q = m2.cells
    kk = np.arange(c1 - c0 + 1, dtype=np.int64)[:, None, None] * n2
    cells = np.concatenate([q[None] + kk, q[None] + kk + n2], axis=2).reshape(-1, 8)
    sub = Mesh(points=pts, cells=cells.astype(np.int64), dim=3)
    off = n0 * n2                                 # sub-mesh id + off = global id
    nc = len(sub.cells)  # large slabs: row ranges of ~0.5M cells (bit-identical, assemble_q1_rows)
    mat = assemble_q1(sub) if nc <= (1 << 21) else assemble_q1_rows(sub, slabs=-(-nc // (1 << 19)))
    ff = _conserved(np.array([1.4]), np.array([[3.0, 0.0, 0.0]]), np.array([1.0]), gas)[0]
    bc = _slip_inflow_bc(sub, lambda X: X[..., 0] < 1e-9, lambda X: X[..., 0] > 4.0 - 1e-9, ff)
    ip, ix = mat.indptr, mat.indices

    def entries(rows):  # CSR positions of the given sub-mesh rows, row by row
        cnt = ip[rows + 1] - ip[rows]
        first = np.repeat(ip[rows] - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
        return first + np.arange(int(cnt.sum()), dtype=np.int64), cnt

    own = np.arange(a - off, b - off, dtype=np.int64)
    sel, own_cnt = entries(own)
    cols_own = ix[sel] + off
    ghosts = np.unique(cols_own[(cols_own < a) | (cols_own >= b)])
    gl = ghosts - off
    gsel, g_cnt = entries(gl)
    gcols = ix[gsel] + off
    keep = ((gcols >= a) & (gcols < b)) | np.isin(gcols, ghosts)
    g_rows = np.repeat(np.arange(len(gl)), g_cnt)
    g_card = np.bincount(g_rows[keep], minlength=len(gl))
    rowptr = np.concatenate([[0], np.cumsum(np.concatenate([own_cnt, g_card]))]).astype(np.int64)
    loc = np.concatenate([own, gl])
    # global pad width and most frequent cardinality (stepper.py:128-131) of the
    # extruded pattern: a node's 3D card is its 2D card times 3 (2 at z = 0, 1)
    card2 = _q1_cardinality(m2)
    hist = np.zeros(3 * int(card2.max()) + 1, dtype=np.int64)
    np.add.at(hist, 3 * card2, max(nz - 1, 0))
    np.add.at(hist, 2 * card2, 2)
    lm = LocalMatrices(n_global=N, dim=3, pad_width=int(np.flatnonzero(hist).max()),
                       standard_card=int(np.argmax(hist)), rank=rank, nranks=nranks, ranges=ranges,
                       ghost_gid=ghosts.astype(np.int64), rowptr=rowptr,
                       col_gid=np.concatenate([cols_own, gcols[keep]]).astype(np.int64),
                       m=np.concatenate([mat.m[sel], mat.m[gsel][keep]]),
                       c=np.concatenate([mat.c[sel], mat.c[gsel][keep]]),
                       m_lumped=mat.m_lumped[loc], inv_m=mat.inv_m[loc],
                       full_card=(ip[loc + 1] - ip[loc]).astype(np.int32))

    def owned(ids):
        g = np.asarray(ids, dtype=np.int64) + off
        return (g >= a) & (g < b), g

    inflow = slip = normals = None
    if bc.inflow_nodes is not None:
        k_in, g = owned(bc.inflow_nodes)
        inflow = g[k_in] if k_in.any() else None
    if bc.slip_nodes is not None:
        k_s, g = owned(bc.slip_nodes)
        if k_s.any():
            slip, normals = g[k_s], bc.slip_normals[k_s]
    bcl = BoundaryConditions(inflow_nodes=inflow, farfield=ff, slip_nodes=slip, slip_normals=normals)
    return LocalProblem("c4-mach3-cylinder", lm, np.tile(ff, (b - a, 1)), c_cfl=0.9, steps=steps,
                        boundary=bcl)


def random_state(rng, n: int, dim: int = 2) -> np.ndarray:
    """Seeded admissible random field (the reference's test fixture, test_stepper.py:15-21)."""
    U = np.zeros((n, dim + 2))
    U[:, 0] = 1.0 + 0.5 * rng.random(n)
    U[:, 1:-1] = rng.normal(0.0, 0.3, (n, dim)) * U[:, 0:1]
    p = 0.5 + rng.random(n)
    U[:, -1] = p / 0.4 + 0.5 * (U[:, 1:-1] ** 2).sum(axis=1) / U[:, 0]
    return U


def _reduced_points(mesh: Mesh) -> np.ndarray:
    """One representative point per solver node (the last periodic copy wins)."""
    pts = np.zeros((mesh.n_nodes, mesh.dim))
    pts[mesh.reduced_index] = mesh.points
    return pts


def periodic_smooth(n: int = 32, refine: int = 0, velocity=(1.0, 0.5), gas: GasConstants = AIR,
                    steps: int = 0) -> ProblemSetup:
    """Density wave advected through the periodic unit square at constant
    velocity and pressure, with its exact solution (reference problems.py:84-121)."""
    n = n * (2 ** refine)
    mesh = rectangle_mesh(n, n, periodic=(True, True))
    v = np.asarray(velocity, dtype=np.float64)

    def exact(points, t):
        rho = 1.0 + 0.3 * np.sin(2.0 * np.pi * (points[:, 0] - v[0] * t)) * np.sin(
            2.0 * np.pi * (points[:, 1] - v[1] * t))
        U = np.zeros((len(points), 4))
        U[:, 0] = rho
        U[:, 1] = rho * v[0]
        U[:, 2] = rho * v[1]
        U[:, 3] = 1.0 / gas.gm1 + 0.5 * rho * (v @ v)
        return U

    U0 = exact(_reduced_points(mesh), 0.0)
    return ProblemSetup("periodic-smooth", assemble_q1(mesh), U0, None, c_cfl=0.9, steps=steps, mesh=mesh,
                        exact=exact)


def sod1d(n: int = 100, refine: int = 0, gas: GasConstants = AIR, steps: int = 0) -> ProblemSetup:
    """Shock tube on a y-periodic strip of n x 1 quads (reference problems.py:124-137)."""
    n = n * (2 ** refine)
    mesh = rectangle_mesh(n, 1, (0.0, 1.0), (0.0, 1.0 / n), periodic=(False, True))
    left = _reduced_points(mesh)[:, 0] < 0.5
    U0 = np.zeros((mesh.n_nodes, 4))
    U0[:, 0] = np.where(left, 1.0, 0.125)
    U0[:, 3] = np.where(left, 1.0, 0.1) / gas.gm1
    return ProblemSetup("sod1d", assemble_q1(mesh), U0, None, c_cfl=0.9, steps=steps, mesh=mesh)


# problem names the command line accepts (cli.py): the BASELINE.json configs and
# the reference's two analytic 2D set-ups
PROBLEMS = ("c1", "c2", "c3", "c4", "c5", "c3m", "c4m", "c5m", "periodic-smooth", "sod1d")


def make_problem(name: str, refine: int = 0, scale: str = "full", gas: GasConstants = AIR) -> ProblemSetup:
    """Problem factory of the command line (reference problems.py:140-146)."""
    if name == "periodic-smooth":
        return periodic_smooth(refine=refine, gas=gas)
    if name == "sod1d":
        return sod1d(refine=refine, gas=gas)
    if name in PROBLEMS:
        return make_config(name, scale=scale, gas=gas)
    raise ValueError(f"unknown problem {name!r}")


def make_config(name: str, scale: str = "full", gas: GasConstants = AIR) -> ProblemSetup:
    """BASELINE.json configs by name; scale='small' gives oracle-sized instances."""
    small = scale == "small"
    if name == "c1":
        return isentropic_vortex(32 if small else 128, gas=gas)
    if name == "c2":
        return mach3_disc(50 if small else 550, gas=gas)
    if name == "c3":
        return sod_box(*((31, 7, 7) if small else (511, 127, 127)), gas=gas)
    if name == "c5":
        return periodic_fourier_box(12 if small else 320, gas=gas)
    if name == "c4":  # ~67M nodes: the 8-GPU configuration
        return mach3_cylinder(*((20, 6) if small else (255, 255)), gas=gas)
    if name == "c4m":  # single-GPU C4-shaped instance (~2.1M nodes)
        return mach3_cylinder(*((20, 6) if small else (100, 50)), gas=gas)
    if name == "c3m":  # mid-size Sod box (1.05M nodes) for quick measurements
        return sod_box(*((31, 7, 7) if small else (255, 63, 63)), gas=gas)
    if name == "c5m":  # mid-size 3D instance for quick measurements
        return periodic_fourier_box(12 if small else 160, gas=gas)
    raise ValueError(f"unknown config {name!r}")

"""Offline inputs: Q1 assembly and the BASELINE config generators."""

import os
import sys

import numpy as np
import pytest

from paper_2007_00094_b200 import problems as P

REF_SRC = "/root/reference/pkg/src"


def _check_matrices(mat):
    n = mat.n
    card = np.diff(mat.indptr)
    assert (card >= 1).all()
    rows = np.repeat(np.arange(n), card)
    # sorted, duplicate-free columns and a structurally symmetric pattern
    key = rows * n + mat.indices
    assert (np.diff(key) > 0).all()
    keyT = np.sort(mat.indices * n + rows)
    assert np.array_equal(key, keyT)
    # m symmetric, lumped mass positive, rows of c sum to zero (partition of unity)
    order = np.argsort(keyT.argsort())
    assert (mat.m_lumped > 0).all()
    csum = np.add.reduceat(mat.c, mat.indptr[:-1], axis=0)
    assert np.abs(csum).max() < 1e-12 * max(1.0, np.abs(mat.c).max())
    assert np.allclose(mat.inv_m, 1.0 / mat.m_lumped, rtol=0, atol=0)


@pytest.mark.parametrize("maker", [
    lambda: P.isentropic_vortex(16).matrices,
    lambda: P.mach3_disc(20, seed=1).matrices,
    lambda: P.sod_box(7, 3, 3, seed=2).matrices,
    lambda: P.periodic_fourier_box(5).matrices,
    lambda: P.mach3_cylinder(10, 3, seed=3).matrices,
])
def test_assembly_invariants(maker):
    _check_matrices(maker())


def test_total_mass_equals_domain_measure():
    mat = P.isentropic_vortex(16).matrices
    assert abs(mat.m_lumped.sum() - 100.0) < 1e-11
    mat = P.sod_box(7, 3, 3, jitter=0.2, seed=1).matrices
    assert abs(mat.m_lumped.sum() - 0.0625) < 1e-14


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")
def test_assembly_matches_reference_2d():
    sys.path.insert(0, REF_SRC)
    from eulerflow import assembly, mesh
    rm = mesh.rectangle_mesh(6, 5, x_range=(0, 2), y_range=(-1, 1), periodic=(False, True))
    ref = assembly.assemble(rm)
    ours = P.assemble_q1(P.Mesh(points=rm.points, cells=rm.cells, dim=2, reduced_index=rm.reduced_index))
    assert np.array_equal(ref.indptr, ours.indptr) and np.array_equal(ref.indices, ours.indices)
    assert np.allclose(ref.m, ours.m, rtol=1e-13, atol=1e-15)
    assert np.allclose(ref.c, ours.c, rtol=1e-13, atol=1e-15)
    assert np.allclose(ref.m_lumped, ours.m_lumped, rtol=1e-13)


def test_c2_boundary_classification():
    ps = P.mach3_disc(20, seed=1)
    bc = ps.boundary
    x = np.zeros(ps.matrices.n)
    x[:] = ps.mesh.points[:, 0]
    assert (np.abs(x[bc.inflow_nodes]) < 1e-12).all()
    assert not np.intersect1d(bc.inflow_nodes, bc.slip_nodes).size
    assert np.allclose(np.linalg.norm(bc.slip_normals, axis=1), 1.0)
    assert np.allclose(bc.farfield, [1.4, 4.2, 0.0, 1.0 / 0.4 + 0.5 * 1.4 * 9.0])


def test_vortex_initial_state_is_admissible_and_far_field_matches():
    ps = P.isentropic_vortex(32)
    U = ps.U0
    eps = U[:, -1] - 0.5 * (U[:, 1:-1] ** 2).sum(axis=1) / U[:, 0]
    assert (U[:, 0] > 0).all() and (eps > 0).all()
    corner = np.argmax(np.abs(ps.mesh.points).sum(axis=1))
    assert np.allclose(U[corner], ps.boundary.farfield, rtol=1e-6)


def test_c4_extruded_cylinder_geometry():
    """C4: [0,4]x[0,1]^2 minus the cylinder r=0.1 (polygonal O-grid boundary),
    stencils of 27 points with 33 at the O-grid junctions."""
    ps = P.mach3_cylinder(20, 4, seed=3)
    mat = ps.matrices
    vol = mat.m_lumped.sum()
    assert abs(vol - (4.0 - np.pi * 0.01)) < 2e-3
    card = np.diff(mat.indptr)
    assert np.bincount(card).argmax() == 27 and card.max() <= 33
    assert len(ps.boundary.inflow_nodes) > 0 and len(ps.boundary.slip_nodes) > 0
    assert np.allclose(np.linalg.norm(ps.boundary.slip_normals, axis=1), 1.0)


@pytest.mark.parametrize("slabs", [1, 3, 7])
def test_row_range_assembly_is_bitwise_identical(slabs):
    """assemble_q1_rows (used for the full C3 box) equals assemble_q1 bit for bit."""
    meshes = [P.box_mesh(9, 5, 4, jitter=0.2, seed=3), P.extrude(P.disc_channel_mesh(10), 3), P.disc_channel_mesh(20),
              P.rectangle_mesh(7, 5)]
    for mesh in meshes:
        a = P.assemble_q1(mesh)
        b = P.assemble_q1_rows(mesh, slabs=slabs)
        for f in ("indptr", "indices", "m", "c", "m_lumped", "inv_m"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f

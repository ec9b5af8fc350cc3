"""Snapshot output and the perf report: the reference's
`output.schlieren` / `output.write_vtk` and `perf.format_table` API.  The VTK
file is compared with the reference's own writer on the same mesh and state
when the reference tree is present (build container only)."""

import os
import sys

import numpy as np
import pytest

from paper_2007_00094_b200 import output, perf
from paper_2007_00094_b200 import problems as P

REF_SRC = "/root/reference/pkg/src"


def test_schlieren_constant_and_range():
    ps = P.isentropic_vortex(16)
    U = np.tile(ps.U0[0], (ps.matrices.n, 1))
    assert np.array_equal(output.schlieren(U, ps.matrices), np.ones(ps.matrices.n))
    s = output.schlieren(ps.U0, ps.matrices)
    assert s.min() > 0.0 and s.max() <= 1.0 and abs(s.min() - np.exp(-10.0)) < 1e-12


@pytest.mark.parametrize("maker", [lambda: P.isentropic_vortex(8), lambda: P.sod_box(3, 2, 2, seed=1)])
def test_write_vtk_layout(tmp_path, maker):
    ps = maker()
    path = tmp_path / "snap.vtk"
    output.write_vtk(str(path), ps.mesh, ps.U0, ps.matrices)
    txt = path.read_text().splitlines()
    assert txt[0] == "# vtk DataFile Version 3.0" and txt[3] == "DATASET UNSTRUCTURED_GRID"
    npts = len(ps.mesh.points)
    assert txt[4] == f"POINTS {npts} double"
    assert f"POINT_DATA {npts}" in txt and "SCALARS schlieren double" in txt


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")
def test_write_vtk_matches_reference_writer(tmp_path):
    sys.path.insert(0, REF_SRC)
    from eulerflow import output as r_output  # noqa: E402

    ps = P.mach3_disc(10, seed=3)
    a, b = tmp_path / "ours.vtk", tmp_path / "ref.vtk"
    U = ps.U0 * (1.0 + 0.01 * np.sin(np.arange(ps.matrices.n)))[:, None]
    output.write_vtk(str(a), ps.mesh, U, ps.matrices)
    r_output.write_vtk(str(b), ps.mesh, U, ps.matrices)
    assert a.read_text() == b.read_text()


def test_perf_table_lists_model_and_kernels():
    txt = perf.format_table(3, config="c5m")
    assert "dim=3" in txt and "k_edge_visc" in txt
    t = perf.predict_traffic(3, 27)
    assert abs(sum(t[k] for k in ("step0", "step1", "step2", "step3", "step4", "step5", "step6")) -
               39.167) < 1e-3

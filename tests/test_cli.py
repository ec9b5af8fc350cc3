"""Command line and run configuration (the reference's pkg/tests/test_output_cli.py:104-170)."""

import os

import numpy as np
import pytest

from paper_2007_00094_b200 import problems
from paper_2007_00094_b200.cli import build_parser, main
from paper_2007_00094_b200.config import RunConfig, parse_config_file


def test_config_file_parsing(tmp_path):
    f = tmp_path / "run.cfg"
    f.write_text("problem = sod1d\nrefine=1  # one uniform refinement\nt-final = 0.05\nranks = 2\n"
                 "overlap = off\nscale = small\n\n")
    cfg = parse_config_file(str(f))
    assert (cfg.problem, cfg.refine, cfg.t_final, cfg.ranks, cfg.overlap, cfg.scale) == (
        "sod1d", 1, 0.05, 2, False, "small")


def test_config_rejects_bad_input(tmp_path):
    bad = tmp_path / "bad.cfg"
    bad.write_text("no_such_key = 1\n")
    with pytest.raises(ValueError):
        parse_config_file(str(bad))
    nokv = tmp_path / "nokv.cfg"
    nokv.write_text("problem sod1d\n")
    with pytest.raises(ValueError):
        parse_config_file(str(nokv))
    for kw in ({"problem": "nope"}, {"c_cfl": 2.0}, {"c_cfl": 0.0}, {"ranks": 0}, {"t_final": 0.0},
               {"output_every": -1}, {"limiter_passes": -1}, {"scale": "huge"}, {"backend": "cpu"}):
        with pytest.raises(ValueError):
            RunConfig(**kw).validate()


def test_parser_exposes_documented_flags():
    text = build_parser().format_help()
    for flag in ["--problem", "--refine", "--t-final", "--cfl", "--limiter-passes", "--newton-steps",
                 "--lanes", "--workers", "--ranks", "--no-overlap", "--output-every", "--output-dir",
                 "--perf", "--scale", "--backend"]:
        assert flag in text


def test_cli_rejects_bad_cfl(capsys):
    assert main(["--problem", "sod1d", "--cfl", "1.7", "--t-final", "0.01"]) == 1
    assert "error" in capsys.readouterr().err


def test_problem_factory_names():
    for name in ("periodic-smooth", "sod1d", "c1", "c2", "c3", "c4", "c5"):
        s = problems.make_problem(name, scale="small")
        U = s.U0
        assert U.shape == (s.matrices.n, s.matrices.dim + 2)
        eps = U[:, -1] - 0.5 * (U[:, 1:-1] ** 2).sum(axis=1) / U[:, 0]
        assert (U[:, 0] > 0).all() and (eps > 0).all()
    with pytest.raises(ValueError):
        problems.make_problem("bogus")


def test_periodic_smooth_exact_at_zero_matches_initial_state():
    s = problems.periodic_smooth(n=8)
    pts = np.zeros((s.mesh.n_nodes, 2))
    pts[s.mesh.reduced_index] = s.mesh.points
    assert np.array_equal(s.exact(pts, 0.0), s.U0)
    assert s.matrices.n == 64  # 8 x 8 periodic


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path):
    out = tmp_path / "out"
    rc = main(["--problem", "sod1d", "--t-final", "0.01", "--cfl", "0.5", "--ranks", "2", "--workers", "2",
               "--output-dir", str(out), "--output-every", "2", "--perf"])
    assert rc == 0
    files = os.listdir(out)
    for f in ("sod1d_0000.vtk", "sod1d_0002.vtk", "sod1d_final.vtk", "perf.csv"):
        assert f in files
    rows = (out / "perf.csv").read_text().splitlines()
    assert len(rows) == 1 + 7 + 1

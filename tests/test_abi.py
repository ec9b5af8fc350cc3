"""The C-ABI library loads and exports every symbol include/ef_b200.h declares
(no GPU needed: nothing here launches a kernel)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ef_b200.h")


@pytest.fixture(scope="module")
def lib_path():
    from paper_2007_00094_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2007_00094_b200", "csrc")], check=True)
    return _lib.LIB_PATH


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ef_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_solver_surface():
    names = declared_symbols()
    for required in ("ef_create", "ef_destroy", "ef_set_state", "ef_get_state", "ef_euler_step",
                     "ef_ssp_rk3_step", "ef_last_error", "ef_bad_node", "ef_phase_times",
                     "ef_debug_fetch", "ef_pow_host"):
        assert required in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header(lib_path):
    from paper_2007_00094_b200 import _lib
    assert set(declared_symbols()) == set(_lib.SIGNATURES)
    _lib.load()


def test_host_pow_equals_oracle_pow(lib_path):
    import oracle as O
    from paper_2007_00094_b200 import shared_pow
    rng = np.random.default_rng(3)
    x = np.concatenate([np.exp(rng.uniform(-50, 50, 50000)), rng.uniform(0, 4, 50000)])
    for y in (1 / 2.4, -1.4, 2.4, 1.4, 2.8 / 0.4, -(0.4 / 2.8)):
        assert np.array_equal(shared_pow(x, y), O.shared_pow(x, y))


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: a missing CUDA library is a hard error."""
    code = ("import os, sys; os.environ['EF_B200_LIB'] = sys.argv[1]\n"
            "from paper_2007_00094_b200 import _lib\n"
            "try:\n    _lib.load()\nexcept RuntimeError as e:\n    print('raised', e)\n")
    out = subprocess.run(["python", "-c", code, str(tmp_path / "nope.so")], capture_output=True, text=True,
                         cwd=ROOT)
    assert "raised" in out.stdout


def test_bad_parameters_raise_before_device_use():
    from paper_2007_00094_b200 import Solver, problems
    mat = problems.assemble_q1(problems.rectangle_mesh(4, 4, periodic=(True, True)))
    for kw in (dict(c_cfl=0.0), dict(c_cfl=1.5), dict(limiter_passes=-1)):
        with pytest.raises(ValueError):
            Solver(mat, **kw)

"""ctypes binding of libef_b200.so (the C-ABI declared in include/ef_b200.h).

There is no fallback: if the CUDA library is missing or no GPU is visible,
calls fail loudly.  Build it with `python -c "import __graft_entry__ as g; g.build()"`
(or `make -C paper_2007_00094_b200/csrc`).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EF_B200_LIB") or os.path.join(_HERE, "libef_b200.so")

EF_OK, EF_ERR_ARG, EF_ERR_INADMISSIBLE, EF_ERR_TAU_UNBOUNDED, EF_ERR_CUDA, EF_ERR_NCCL = range(6)

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_d = ctypes.c_double


class EfMatrices(ctypes.Structure):
    _fields_ = [("n", _i64), ("dim", _i32), ("indptr", _p), ("indices", _p), ("m", _p), ("c", _p),
                ("m_lumped", _p), ("inv_m", _p)]


class EfParams(ctypes.Structure):
    _fields_ = [("gamma", _d), ("gm1", _d), ("gp1_inv", _d), ("gm1_over_2g", _d),
                ("two_g_over_gm1", _d), ("c_cfl", _d), ("limiter_passes", _i32),
                ("newton_steps", _i32), ("overlap", _i32)]


class EfBoundary(ctypes.Structure):
    _fields_ = [("n_inflow", _i64), ("inflow", _p), ("farfield", _p), ("n_slip", _i64),
                ("slip", _p), ("slip_normals", _p)]


class EfLocalMatrices(ctypes.Structure):
    _fields_ = [("n_global", _i64), ("dim", _i32), ("pad_width", _i32), ("standard_card", _i32),
                ("n_owned", _i64), ("n_ghost", _i64), ("ghost_gid", _p), ("rowptr", _p), ("col_gid", _p),
                ("m", _p), ("c", _p), ("m_lumped", _p), ("inv_m", _p), ("full_card", _p)]


class EfDist(ctypes.Structure):
    _fields_ = [("rank", _i32), ("nranks", _i32), ("device", _i32), ("cm_perm", _p), ("ranges", _p),
                ("nccl_id", _p), ("stream", _p)]


# every symbol include/ef_b200.h declares, with (restype, argtypes)
SIGNATURES = {
    "ef_create": (_i32, [ctypes.POINTER(EfMatrices), ctypes.POINTER(EfParams),
                         ctypes.POINTER(EfBoundary), ctypes.POINTER(EfDist), ctypes.POINTER(_p)]),
    "ef_destroy": (_i32, [_p]),
    "ef_eval_dij": (_i32, [ctypes.POINTER(EfParams), _i32, _i64, _p, _p, _p, _p, _p, _p]),
    "ef_eval_limiter": (_i32, [ctypes.POINTER(EfParams), _i32, _i64, _p, _p, _p, _p]),
    "ef_eval_arith": (_i32, [_i64, _p, _p, _p]),
    "ef_set_state": (_i32, [_p, _p]),
    "ef_get_state": (_i32, [_p, _p]),
    "ef_euler_step": (_i32, [_p, _i32, _d, _d, ctypes.POINTER(_d)]),
    "ef_ssp_rk3_step": (_i32, [_p, _i32, _d, _d, ctypes.POINTER(_d)]),
    "ef_ssp_rk3_step_async": (_i32, [_p, _i32, _d, _d]),
    "ef_sync": (_i32, [_p, ctypes.POINTER(_d)]),
    "ef_bad_node": (_i64, [_p]),
    "ef_last_error": (ctypes.c_char_p, []),
    "ef_kernel_launches": (_i64, []),
    "ef_enable_timers": (_i32, [_p, _i32]),
    "ef_enable_graphs": (_i32, [_p, _i32]),
    "ef_set_uniform": (_i32, [_p, _i32]),
    "ef_phase_times": (_i32, [_p, _p]),
    "ef_counters": (_i32, [_p, _p]),
    "ef_info": (_i32, [_p, _p]),
    "ef_debug_fetch": (_i32, [_p, _i32, _i32, _p]),
    "ef_local_gids": (_i32, [_p, _p]),
    "ef_pow_host": (None, [_p, _d, _p, _i64]),
    "ef_pow_device": (_i32, [_p, _d, _p, _i64]),
    "ef_pow_bound_device": (_i32, [_p, _d, _p, _i64]),
    "ef_state_device_ptr": (_i32, [_p, ctypes.POINTER(_p), ctypes.POINTER(_i64)]),
    "ef_nccl_unique_id": (_i32, [_p]),
    "ef_group_create": (_i32, [_p, _i32, ctypes.POINTER(_p)]),
    "ef_group_destroy": (_i32, [_p]),
    "ef_group_set_state": (_i32, [_p, _p]),
    "ef_group_get_state": (_i32, [_p, _p]),
    "ef_group_euler_step": (_i32, [_p, _i32, _d, _d, ctypes.POINTER(_d)]),
    "ef_group_ssp_rk3_step": (_i32, [_p, _i32, _d, _d, ctypes.POINTER(_d)]),
    "ef_plan_build": (_i32, [ctypes.POINTER(EfMatrices), ctypes.POINTER(EfDist), ctypes.POINTER(_p)]),
    "ef_plan_destroy": (_i32, [_p]),
    "ef_plan_sizes": (_i32, [_p, _p]),
    "ef_plan_rows": (_i64, [_p, _i32, _i32, _p, _i64]),
    "ef_plan_build_local": (_i32, [ctypes.POINTER(EfLocalMatrices), ctypes.POINTER(EfDist), ctypes.POINTER(_p)]),
    "ef_create_local": (_i32, [ctypes.POINTER(EfLocalMatrices), ctypes.POINTER(EfParams),
                               ctypes.POINTER(EfBoundary), ctypes.POINTER(EfDist), ctypes.POINTER(_p)]),
    "ef_set_state_owned": (_i32, [_p, _p]),
    "ef_get_state_owned": (_i32, [_p, _p]),
    "ef_group_set_state_owned": (_i32, [_p, _p]),
    "ef_group_get_state_owned": (_i32, [_p, _p]),
}

_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension {LIB_PATH} is not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().ef_last_error()
    return msg.decode() if msg else ""

"""ctypes binding of libcvxreg_b200.so (the C ABI in include/cvxreg_b200.h).

The library is the product: there is no CPU fallback. If the shared object is
missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CRB_LIB") or os.path.join(PKG, "libcvxreg_b200.so")

CR_STATUS = {0: "CR_OK", 1: "CR_EINVAL", 2: "CR_ENOMEM", 3: "CR_ECUDA", 4: "CR_ENCCL",
             5: "CR_ENONFINITE", 6: "CR_ESTATE"}

_P = C.POINTER(C.c_double)


class PapgConfigC(C.Structure):
    _fields_ = [
        ("gamma", C.c_double), ("B_theta", C.c_double),
        ("adaptive_B_theta", C.c_int32), ("max_restarts", C.c_int32),
        ("gap_norm_tol", C.c_double), ("infeas_norm_tol", C.c_double),
        ("max_iters", C.c_int64), ("max_seconds", C.c_double),
        ("inner_tol_floor", C.c_double), ("final_resolve_tol", C.c_double),
        ("record_history", C.c_int32), ("use_momentum", C.c_int32),
        ("sigma_C", C.c_double), ("graph_iters", C.c_int32), ("workers", C.c_int32),
    ]


class PapgResultC(C.Structure):
    _fields_ = [
        ("iters", C.c_int64), ("reason", C.c_int32), ("restarts", C.c_int32),
        ("saturated", C.c_int32), ("sigma_iters", C.c_int32),
        ("sigma_converged", C.c_int32), ("history_truncated", C.c_int32),
        ("g_final", C.c_double), ("delta_estimate", C.c_double), ("sigma_C", C.c_double),
        ("L_g", C.c_double), ("B_theta", C.c_double), ("wall_seconds", C.c_double),
        ("sigma_seconds", C.c_double), ("loop_seconds", C.c_double),
        ("last_gap_norm", C.c_double), ("last_infeas_norm", C.c_double),
    ]


class AlccConfigC(C.Structure):
    _fields_ = [
        ("mu1", C.c_double), ("tau1_scale", C.c_double), ("alpha1_scale", C.c_double),
        ("c", C.c_double), ("kappa", C.c_double), ("max_outer", C.c_int64),
        ("mapg_cap", C.c_int64), ("infeas_norm_tol", C.c_double), ("gap_norm_tol", C.c_double),
        ("max_seconds", C.c_double), ("record_history", C.c_int32), ("pad_", C.c_int32),
        ("sigma_A1", C.c_double), ("sigma_A2", C.c_double), ("Bbar_y", C.c_double),
        ("Bbar_xi", C.c_double),
    ]


class AlccResultC(C.Structure):
    _fields_ = [
        ("outer_iters", C.c_int64), ("mapg_iters_total", C.c_int64), ("reason", C.c_int32),
        ("hit_cap_any", C.c_int32), ("sigma_A1_iters", C.c_int32), ("sigma_A2_iters", C.c_int32),
        ("certified_gap", C.c_double), ("infeas_raw", C.c_double), ("gap_raw", C.c_double),
        ("objective", C.c_double), ("wall_seconds", C.c_double), ("sigma_A1", C.c_double),
        ("sigma_A2", C.c_double), ("sigma_seconds", C.c_double), ("mapg_seconds", C.c_double),
        ("launches", C.c_int64),
    ]


HISTORY_CAP = 4000000  # CR_HISTORY_CAP (include/cvxreg_b200.h)

# every symbol declared in include/cvxreg_b200.h
EXPORTS = [
    "cr_create", "cr_destroy", "cr_last_error", "cr_status_string", "cr_nccl_unique_id",
    "cr_attach_nccl", "cr_exchange_len", "cr_sigma_C", "cr_papg_begin", "cr_papg_iterate",
    "cr_iter_local", "cr_exchange_get", "cr_exchange_put", "cr_iter_finish", "cr_papg_finish",
    "cr_papg_solve", "cr_get_theta", "cr_get_rows", "cr_get_theta_rows", "cr_get_rows_window",
    "cr_last_timing", "cr_last_sweep_times", "cr_last_exchange_seconds", "cr_time_sweep",
    "cr_sweep_variant", "cr_papg_begin_resume", "cr_set_observations", "cr_infeasibility",
    "cr_duality_gap", "cr_evaluate_estimator", "cr_repair_feasibility",
    "cr_gen_instance", "cr_prepare_problem", "cr_certificate", "cr_momentum_next",
    "cr_sigma_A", "cr_alcc_solve", "cr_alcc_multiplier", "cr_time_penalty_sweep",
    "cr_set_partition", "cr_partition_stats", "cr_sweep_store_count",
    "cr_set_canonical_blocks", "cr_canonical_blocks",
]

_lib = None


class NativeError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{CR_STATUS.get(status, status)}: {msg}")
        self.status = status


def load():
    """Load the shared library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_1407_7220_b200.build`")
    L = C.CDLL(LIB_PATH)
    i64, i32, u64, d, vp = C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_void_p
    st = C.c_int
    sig = {
        "cr_create": (st, [_P, _P, i64, i64, d, C.c_int, i64, i64, C.POINTER(vp)]),
        "cr_destroy": (None, [vp]),
        "cr_last_error": (C.c_char_p, [vp]),
        "cr_status_string": (C.c_char_p, [st]),
        "cr_nccl_unique_id": (st, [C.c_char_p]),
        "cr_attach_nccl": (st, [vp, C.c_char_p, C.c_int, C.c_int]),
        "cr_exchange_len": (i64, [vp]),
        "cr_set_canonical_blocks": (st, [vp, i32]),
        "cr_canonical_blocks": (st, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
        "cr_sigma_C": (st, [vp, d, i32, _P, C.POINTER(i32), C.POINTER(i32)]),
        "cr_papg_begin": (st, [vp, C.POINTER(PapgConfigC), _P]),
        "cr_papg_iterate": (st, [vp, i64, C.POINTER(i64), C.POINTER(i32)]),
        "cr_iter_local": (st, [vp]),
        "cr_exchange_get": (st, [vp, _P]),
        "cr_exchange_put": (st, [vp, _P]),
        "cr_iter_finish": (st, [vp, C.POINTER(i32)]),
        "cr_papg_finish": (st, [vp, C.POINTER(PapgResultC), _P, _P, _P]),
        "cr_papg_solve": (st, [vp, C.POINTER(PapgConfigC), _P, C.POINTER(PapgResultC), _P, _P, _P]),
        "cr_get_theta": (st, [vp, _P]),
        "cr_get_rows": (st, [vp, _P]),
        "cr_get_theta_rows": (st, [vp, i64, i64, _P]),
        "cr_get_rows_window": (st, [vp, i64, i64, _P]),
        "cr_last_timing": (st, [vp, _P, C.POINTER(i64), _P]),
        "cr_last_sweep_times": (st, [vp, _P, i64, C.POINTER(i64)]),
        "cr_last_exchange_seconds": (st, [vp, _P]),
        "cr_time_sweep": (st, [vp, i32, _P]),
        "cr_sweep_variant": (i32, [vp]),
        "cr_papg_begin_resume": (st, [vp, C.POINTER(PapgConfigC)]),
        "cr_set_observations": (st, [vp, _P]),
        "cr_infeasibility": (st, [vp, _P, _P, _P]),
        "cr_duality_gap": (st, [vp, _P, _P, _P]),
        "cr_evaluate_estimator": (st, [vp, _P, _P, _P, i64, _P]),
        "cr_repair_feasibility": (st, [vp, _P, _P, _P]),
        "cr_gen_instance": (st, [i32, i64, i64, d, u64, i64, _P, _P]),
        "cr_prepare_problem": (st, [_P, _P, i64, i64, d, _P, _P, _P, _P, _P]),
        "cr_certificate": (None, [d, d, d, d, _P]),
        "cr_momentum_next": (d, [d]),
        "cr_sigma_A": (st, [vp, i32, d, i32, _P, C.POINTER(i32), C.POINTER(i32)]),
        "cr_alcc_solve": (st, [vp, C.POINTER(AlccConfigC), _P, _P, _P, _P, _P,
                               C.POINTER(i64), C.POINTER(AlccResultC)]),
        "cr_alcc_multiplier": (st, [vp, i64, i64, _P]),
        "cr_time_penalty_sweep": (st, [vp, i32, _P]),
        "cr_set_partition": (st, [vp, i64, _P, _P, C.POINTER(AlccConfigC)]),
        "cr_partition_stats": (st, [vp, C.POINTER(i64), _P, _P, _P]),
        "cr_sweep_store_count": (st, [vp, C.POINTER(u64), i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def check(status, handle=None, what=""):
    if status != 0:
        L = load()
        msg = L.cr_last_error(handle).decode() if handle else L.cr_status_string(status).decode()
        raise NativeError(status, f"{what}: {msg}" if what else msg)

"""ctypes wrapper for the CPU restatement -- TEST INFRASTRUCTURE ONLY.

Loads oracle/libcvxreg_oracle.so (built by oracle/Makefile). Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this module; the
product package paper_1407_7220_b200 never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcvxreg_oracle.so")

GEN_KINDS = {
    "quadratic": 0, "exponential": 1, "affine-noiseless": 2, "custom-1d": 3,
    "sqnorm-uniform": 10, "maxaffine-uniform": 11, "lse-uniform": 12,
}
REASONS = {0: "thresholds", 1: "iter_budget", 2: "time_budget", 3: "error"}
REASONS_INV = {v: k for k, v in REASONS.items()}


class CroConfig(C.Structure):
    _fields_ = [
        ("gamma", C.c_double), ("B_theta", C.c_double),
        ("adaptive_B_theta", C.c_int32), ("max_restarts", C.c_int32),
        ("gap_norm_tol", C.c_double), ("infeas_norm_tol", C.c_double),
        ("max_iters", C.c_int64), ("max_seconds", C.c_double),
        ("inner_tol_floor", C.c_double), ("final_resolve_tol", C.c_double),
        ("record_history", C.c_int32), ("use_momentum", C.c_int32),
        ("sigma_C", C.c_double), ("threads", C.c_int32), ("pad_", C.c_int32),
    ]


_P = C.POINTER(C.c_double)


class CroResult(C.Structure):
    _fields_ = [
        ("y", _P), ("xi", _P), ("theta", _P), ("c_eta", _P), ("history", _P),
        ("iters", C.c_int64), ("reason", C.c_int32), ("restarts", C.c_int32),
        ("saturated", C.c_int32), ("sigma_iters", C.c_int32),
        ("sigma_converged", C.c_int32), ("pad_", C.c_int32),
        ("g_final", C.c_double), ("delta_estimate", C.c_double),
        ("sigma_C", C.c_double), ("L_g", C.c_double), ("B_theta", C.c_double),
        ("wall_seconds", C.c_double),
    ]


class CroAlccConfig(C.Structure):
    _fields_ = [
        ("mu1", C.c_double), ("tau1_scale", C.c_double), ("alpha1_scale", C.c_double),
        ("c", C.c_double), ("kappa", C.c_double), ("max_outer", C.c_int64),
        ("mapg_cap", C.c_int64), ("infeas_norm_tol", C.c_double), ("gap_norm_tol", C.c_double),
        ("max_seconds", C.c_double), ("record_history", C.c_int32), ("threads", C.c_int32),
    ]


class CroAlccResult(C.Structure):
    _fields_ = [
        ("y", _P), ("xi", _P), ("multiplier", _P), ("history", _P),
        ("mapg_iters", C.POINTER(C.c_int64)),
        ("outer_iters", C.c_int64), ("mapg_iters_total", C.c_int64),
        ("reason", C.c_int32), ("hit_cap_any", C.c_int32),
        ("certified_gap", C.c_double), ("infeas_raw", C.c_double), ("gap_raw", C.c_double),
        ("objective", C.c_double), ("wall_seconds", C.c_double), ("sigma_A1", C.c_double),
        ("sigma_A2", C.c_double),
    ]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        d, i64, i32, u64 = C.c_double, C.c_int64, C.c_int, C.c_uint64
        L.cro_rng_draws.argtypes = [u64, u64, i64, i32, _P]
        L.cro_rng_draws.restype = u64
        L.cro_gen_instance.argtypes = [i32, i64, i64, d, u64, i64, _P, _P]
        L.cro_prepare.argtypes = [_P, _P, i64, i64, d, _P, _P, _P, _P, _P, _P, _P]
        L.cro_apply_C.argtypes = [_P, i64, i64, _P, _P, _P]
        L.cro_apply_C.restype = None
        L.cro_apply_C_T.argtypes = [_P, i64, i64, _P, _P, _P]
        L.cro_apply_C_T.restype = None
        L.cro_sigma_C.argtypes = [_P, i64, i64, d, i32, _P, C.POINTER(i32), C.POINTER(i32)]
        L.cro_papg.argtypes = [_P, _P, i64, i64, C.POINTER(CroConfig), _P, C.POINTER(CroResult)]
        L.cro_project_nonneg_ball.argtypes = [_P, i64, d]
        L.cro_project_nonneg_ball.restype = None
        L.cro_momentum_next.argtypes = [d]
        L.cro_momentum_next.restype = d
        L.cro_certificate.argtypes = [d, d, d, d, _P]
        L.cro_certificate.restype = None
        L.cro_infeasibility.argtypes = [_P, i64, i64, _P, _P, _P]
        L.cro_infeasibility.restype = None
        L.cro_duality_gap.argtypes = [_P, i64, i64, _P, _P, _P, _P]
        L.cro_duality_gap.restype = None
        L.cro_evaluate_estimator.argtypes = [_P, i64, i64, _P, _P, _P]
        L.cro_evaluate_estimator.restype = d
        L.cro_repair_feasibility.argtypes = [_P, i64, i64, _P, _P, _P]
        L.cro_repair_feasibility.restype = None
        L.cro_sigma_A.argtypes = [_P, i64, i64, i32, d, i32, _P, C.POINTER(i32), C.POINTER(i32)]
        L.cro_alcc.argtypes = [_P, _P, i64, i64, d, d, d, d, d, _P, _P,
                               C.POINTER(CroAlccConfig), C.POINTER(CroAlccResult)]
        L.cro_apply_C_k.argtypes = [_P, i64, i64, i64, _P, _P, _P]
        L.cro_apply_C_k.restype = None
        L.cro_apply_C_T_k.argtypes = [_P, i64, i64, i64, _P, _P, _P]
        L.cro_apply_C_T_k.restype = None
        L.cro_sigma_C_k.argtypes = [_P, i64, i64, i64, d, i32, _P, C.POINTER(i32), C.POINTER(i32)]
        L.cro_papg_k.argtypes = [_P, _P, i64, i64, i64, C.POINTER(CroConfig),
                                 C.POINTER(CroAlccConfig), _P, _P, _P, C.POINTER(CroResult),
                                 C.POINTER(C.c_int64)]
        L.cro_papg_replay.argtypes = [_P, _P, i64, i64, C.POINTER(CroConfig),
                                      C.POINTER(C.c_int64), i64, _P, _P, C.POINTER(CroResult)]
        L.cro_cross_position.argtypes = [i64, i64, i64, i64]
        L.cro_cross_position.restype = i64
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_P) if a is not None else None


def rng_draws(seed, tag, count, kind="uniform"):
    out = np.empty(count, np.float64)
    lib().cro_rng_draws(seed, tag, count, {"uniform": 0, "normal": 1, "raw53": 2}[kind], _p(out))
    return out


def gen_instance(kind, N, n, noise=1.0, seed=1, pieces=0):
    X = np.empty((N, n), np.float64)
    y = np.empty(N, np.float64)
    rc = lib().cro_gen_instance(GEN_KINDS[kind], N, n, noise, seed, pieces, _p(X), _p(y))
    if rc != 0:
        raise ValueError(f"oracle gen_instance failed ({rc})")
    return X, y


@dataclass
class Prepared:
    X: np.ndarray
    ys: np.ndarray
    shift: float
    feas_y: np.ndarray
    feas_xi: np.ndarray
    B_theta: float
    Bbar_y: float
    Bbar_xi: float
    gamma: float
    intercept: float
    slope: np.ndarray


def prepare(X, y, gamma=1e-3):
    X = np.ascontiguousarray(X, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    N, n = X.shape
    ys = np.empty(N)
    shift = np.zeros(1)
    fy = np.empty(N)
    fxi = np.empty(N * n)
    b4 = np.empty(4)
    ic = np.zeros(1)
    sl = np.empty(n)
    rc = lib().cro_prepare(_p(X), _p(y), N, n, gamma, _p(ys), _p(shift), _p(fy), _p(fxi),
                           _p(b4), _p(ic), _p(sl))
    if rc != 0:
        raise ValueError("oracle prepare failed")
    return Prepared(X, ys, float(shift[0]), fy, fxi, b4[0], b4[1], b4[2], b4[3], float(ic[0]), sl)


def apply_C(X, y, xi):
    N, n = X.shape
    out = np.empty(N * (N - 1) + N)
    lib().cro_apply_C(_p(np.ascontiguousarray(X)), N, n, _p(np.ascontiguousarray(y)),
                      _p(np.ascontiguousarray(xi).reshape(-1)), _p(out))
    return out


def apply_C_T(X, theta):
    N, n = X.shape
    oy = np.empty(N)
    oxi = np.empty(N * n)
    lib().cro_apply_C_T(_p(np.ascontiguousarray(X)), N, n, _p(np.ascontiguousarray(theta)),
                        _p(oy), _p(oxi))
    return oy, oxi


def sigma_C(X, tol=1e-6, max_iters=5000):
    X = np.ascontiguousarray(X, np.float64)
    N, n = X.shape
    s = np.zeros(1)
    it = C.c_int(0)
    cv = C.c_int(0)
    rc = lib().cro_sigma_C(_p(X), N, n, tol, max_iters, _p(s), C.byref(it), C.byref(cv))
    if rc != 0:
        raise MemoryError("oracle sigma_C failed")
    return float(s[0]), it.value, bool(cv.value)


@dataclass
class OracleResult:
    y: np.ndarray
    xi: np.ndarray
    theta: np.ndarray | None
    c_eta: np.ndarray | None
    history: np.ndarray
    iters: int
    reason: str
    restarts: int
    saturated: bool
    g_final: float
    delta_estimate: float
    sigma_C: float
    L_g: float
    B_theta: float
    wall_seconds: float
    sigma_iters: int = 0
    extra: dict = field(default_factory=dict)


def papg(X, ys, *, gamma=1e-3, B_theta=0.0, adaptive_B_theta=True, max_restarts=6,
         gap_norm_tol=1e-6, infeas_norm_tol=1e-1, max_iters=100000, max_seconds=7200.0,
         inner_tol_floor=1e-6, final_resolve_tol=1e-10, record_history=True,
         use_momentum=True, sigma_C=0.0, threads=1, theta0=None, want_theta=True,
         want_c_eta=False):
    X = np.ascontiguousarray(X, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    N, n = X.shape
    dim = N * (N - 1) + N
    cfg = CroConfig(gamma, B_theta, int(adaptive_B_theta), max_restarts, gap_norm_tol,
                    infeas_norm_tol, max_iters, max_seconds, inner_tol_floor, final_resolve_tol,
                    int(record_history), int(use_momentum), sigma_C, threads, 0)
    y = np.empty(N)
    xi = np.empty(N * n)
    theta = np.empty(dim) if want_theta else None
    c_eta = np.empty(dim) if want_c_eta else None
    hist = np.zeros((max_iters if record_history else 0, 8))
    res = CroResult()
    res.y, res.xi, res.theta, res.c_eta = _p(y), _p(xi), _p(theta), _p(c_eta)
    res.history = _p(hist) if record_history else None
    t0 = None if theta0 is None else np.ascontiguousarray(theta0, np.float64)
    rc = lib().cro_papg(_p(X), _p(ys), N, n, C.byref(cfg), _p(t0), C.byref(res))
    if rc == -4:
        raise RuntimeError("papg: non-finite dual gradient")
    if rc != 0:
        raise RuntimeError(f"oracle papg failed ({rc})")
    return OracleResult(y, xi.reshape(N, n), theta, c_eta, hist[: res.iters], int(res.iters),
                        REASONS[res.reason], res.restarts, bool(res.saturated), res.g_final,
                        res.delta_estimate, res.sigma_C, res.L_g, res.B_theta, res.wall_seconds,
                        res.sigma_iters)


def papg_replay(X, ys, *, rows=(), gamma=1e-3, B_theta=0.0, adaptive_B_theta=True,
                max_restarts=6, gap_norm_tol=1e-6, infeas_norm_tol=1e-1, max_iters=100000,
                max_seconds=7200.0, inner_tol_floor=1e-6, final_resolve_tol=1e-10,
                record_history=True, use_momentum=True, sigma_C=0.0, threads=1):
    """Memory-light cro_papg (zero start): no N^2 array. theta / c_eta of the
    result hold the cross rows of the points in `rows` (sorted, (len x (N-1)),
    canonical order) followed by the N pos rows."""
    X = np.ascontiguousarray(X, np.float64)
    ys = np.ascontiguousarray(ys, np.float64)
    N, n = X.shape
    sel = np.unique(np.asarray(rows, np.int64))
    cfg = CroConfig(gamma, B_theta, int(adaptive_B_theta), max_restarts, gap_norm_tol,
                    infeas_norm_tol, max_iters, max_seconds, inner_tol_floor, final_resolve_tol,
                    int(record_history), int(use_momentum), sigma_C, threads, 0)
    y = np.empty(N)
    xi = np.empty(N * n)
    theta = np.empty(sel.size * (N - 1) + N)
    c_eta = np.empty(sel.size * (N - 1) + N)
    hist = np.zeros((max_iters if record_history else 0, 8))
    res = CroResult()
    res.y, res.xi, res.theta, res.c_eta = _p(y), _p(xi), None, None
    res.history = _p(hist) if record_history else None
    rc = lib().cro_papg_replay(_p(X), _p(ys), N, n, C.byref(cfg),
                               sel.ctypes.data_as(C.POINTER(C.c_int64)), sel.size, _p(theta),
                               _p(c_eta), C.byref(res))
    if rc == -4:
        raise RuntimeError("papg: non-finite dual gradient")
    if rc != 0:
        raise RuntimeError(f"oracle papg_replay failed ({rc})")
    return OracleResult(y, xi.reshape(N, n), theta, c_eta, hist[: res.iters], int(res.iters),
                        REASONS[res.reason], res.restarts, bool(res.saturated), res.g_final,
                        res.delta_estimate, res.sigma_C, res.L_g, res.B_theta, res.wall_seconds,
                        res.sigma_iters)


def _c(a):
    return np.ascontiguousarray(a, np.float64)


def infeasibility(X, y, xi):
    X = _c(X)
    out = np.empty(2)
    lib().cro_infeasibility(_p(X), X.shape[0], X.shape[1], _p(_c(y)), _p(_c(xi).reshape(-1)), _p(out))
    return float(out[0]), float(out[1])


def duality_gap(X, theta, y, xi):
    X = _c(X)
    out = np.empty(2)
    lib().cro_duality_gap(_p(X), X.shape[0], X.shape[1], _p(_c(theta)), _p(_c(y)),
                          _p(_c(xi).reshape(-1)), _p(out))
    return float(out[0]), float(out[1])


def evaluate_estimator(X, y, xi, xq):
    X = _c(X)
    return lib().cro_evaluate_estimator(_p(X), X.shape[0], X.shape[1], _p(_c(y)),
                                        _p(_c(xi).reshape(-1)), _p(_c(xq)))


def repair_feasibility(X, y, xi):
    X = _c(X)
    out = np.empty(X.shape[0])
    lib().cro_repair_feasibility(_p(X), X.shape[0], X.shape[1], _p(_c(y)), _p(_c(xi).reshape(-1)),
                                 _p(out))
    return out


def project_nonneg_ball(v, radius):
    v = np.array(v, np.float64)
    lib().cro_project_nonneg_ball(_p(v), v.size, radius)
    return v


def momentum_next(t):
    return lib().cro_momentum_next(t)


def certificate(gamma, delta, B_xi, sigma):
    out = np.empty(2)
    lib().cro_certificate(gamma, delta, B_xi, sigma, _p(out))
    return float(out[0]), float(out[1])


def cross_position(N, K, l1, l2):
    r = lib().cro_cross_position(N, K, l1, l2)
    if r < 0:
        raise ValueError("not a cross-block pair")
    return r


def sigma_A(X, which, tol=1e-6, max_iters=5000):
    """operators.cpp:302-339 on op_A1 (which=1) or op_A2 (which=2)."""
    X = _c(X)
    s = np.zeros(1)
    it = C.c_int(0)
    cv = C.c_int(0)
    rc = lib().cro_sigma_A(_p(X), X.shape[0], X.shape[1], which, tol, max_iters, _p(s),
                           C.byref(it), C.byref(cv))
    if rc != 0:
        raise ValueError(f"oracle sigma_A failed ({rc})")
    return float(s[0]), it.value, bool(cv.value)


@dataclass
class AlccResult:
    y: np.ndarray
    xi: np.ndarray
    multiplier: np.ndarray | None
    history: np.ndarray
    mapg_iters: np.ndarray
    outer_iters: int
    mapg_iters_total: int
    reason: str
    hit_cap_any: bool
    certified_gap: float
    infeas_raw: float
    gap_raw: float
    objective: float
    wall_seconds: float
    sigma_A1: float
    sigma_A2: float


def alcc(X, ys, *, gamma, Bbar_y, Bbar_xi, warm_y, warm_xi, sigma_A1=0.0, sigma_A2=0.0,
         mu1=1.0, tau1_scale=1e-2, alpha1_scale=1e-3, c=5.0, kappa=0.5, max_outer=30,
         mapg_cap=200000, infeas_norm_tol=1e-1, gap_norm_tol=1e-6, max_seconds=float("inf"),
         record_history=True, threads=1, want_multiplier=False):
    """alcc_solve (alcc.cpp:193-208) -> alcc_core (alcc.cpp:54-191), standalone mode."""
    X = _c(X)
    ys = _c(ys)
    N, n = X.shape
    cfg = CroAlccConfig(mu1, tau1_scale, alpha1_scale, c, kappa, max_outer, mapg_cap,
                        infeas_norm_tol, gap_norm_tol, max_seconds, int(record_history), threads)
    y = np.empty(N)
    xi = np.empty(N * n)
    mult = np.empty(N * (N - 1)) if want_multiplier else None
    hist = np.zeros((max_outer, 8))
    mi = np.zeros(max_outer, np.int64)
    res = CroAlccResult()
    res.y, res.xi, res.multiplier, res.history = _p(y), _p(xi), _p(mult), _p(hist)
    res.mapg_iters = mi.ctypes.data_as(C.POINTER(C.c_int64))
    rc = lib().cro_alcc(_p(X), _p(ys), N, n, gamma, Bbar_y, Bbar_xi, sigma_A1, sigma_A2,
                        _p(_c(warm_y)), _p(_c(warm_xi).reshape(-1)), C.byref(cfg), C.byref(res))
    if rc == -5:
        raise RuntimeError("mapg: non-finite gradient")
    if rc != 0:
        raise RuntimeError(f"oracle alcc failed ({rc})")
    k = int(res.outer_iters)
    return AlccResult(y, xi.reshape(N, n), mult, hist[:k], mi[:k], k, int(res.mapg_iters_total),
                      REASONS[res.reason], bool(res.hit_cap_any), res.certified_gap,
                      res.infeas_raw, res.gap_raw, res.objective, res.wall_seconds,
                      res.sigma_A1, res.sigma_A2)


def apply_C_k(X, K, y, xi):
    X = _c(X)
    N, n = X.shape
    out = np.empty(N * (N - N // K) + N)
    lib().cro_apply_C_k(_p(X), N, n, K, _p(_c(y)), _p(_c(xi).reshape(-1)), _p(out))
    return out


def apply_C_T_k(X, K, theta):
    X = _c(X)
    N, n = X.shape
    oy = np.empty(N)
    oxi = np.empty(N * n)
    lib().cro_apply_C_T_k(_p(X), N, n, K, _p(_c(theta)), _p(oy), _p(oxi))
    return oy, oxi


def sigma_C_k(X, K, tol=1e-6, max_iters=5000):
    X = _c(X)
    s = np.zeros(1)
    it = C.c_int(0)
    cv = C.c_int(0)
    rc = lib().cro_sigma_C_k(_p(X), X.shape[0], X.shape[1], K, tol, max_iters, _p(s),
                             C.byref(it), C.byref(cv))
    if rc != 0:
        raise MemoryError("oracle sigma_C_k failed")
    return float(s[0]), it.value, bool(cv.value)


INNER_DEFAULTS = dict(mu1=1.0, tau1_scale=1e-2, alpha1_scale=1e-3, c=5.0, kappa=0.5,
                      max_outer=30, mapg_cap=200000, infeas_norm_tol=1e-1, gap_norm_tol=1e-6,
                      max_seconds=float("inf"), record_history=True)


def papg_k(X, ys, K, feas_y, feas_xi, *, inner=None, gamma=1e-3, B_theta=0.0,
           adaptive_B_theta=True, max_restarts=6, gap_norm_tol=1e-6, infeas_norm_tol=1e-1,
           max_iters=100000, max_seconds=7200.0, inner_tol_floor=1e-6, final_resolve_tol=1e-10,
           record_history=True, use_momentum=True, sigma_C=0.0, threads=1, theta0=None,
           want_c_eta=False, inner_threads=1):
    """General-K P-APG(ALCC) (papg.cpp:136-283, dual_gradient :89-132,
    alcc_solve_block alcc.cpp:222-258)."""
    X = _c(X)
    ys = _c(ys)
    N, n = X.shape
    nbar = N // K
    dim = N * (N - nbar) + N
    cfg = CroConfig(gamma, B_theta, int(adaptive_B_theta), max_restarts, gap_norm_tol,
                    infeas_norm_tol, max_iters, max_seconds, inner_tol_floor, final_resolve_tol,
                    int(record_history), int(use_momentum), sigma_C, threads, 0)
    ic = dict(INNER_DEFAULTS)
    ic.update(inner or {})
    icfg = CroAlccConfig(ic["mu1"], ic["tau1_scale"], ic["alpha1_scale"], ic["c"], ic["kappa"],
                         ic["max_outer"], ic["mapg_cap"], ic["infeas_norm_tol"],
                         ic["gap_norm_tol"], ic["max_seconds"], int(ic["record_history"]),
                         inner_threads)
    y = np.empty(N)
    xi = np.empty(N * n)
    theta = np.empty(dim)
    c_eta = np.empty(dim) if want_c_eta else None
    hist = np.zeros((max_iters if record_history else 0, 8))
    res = CroResult()
    res.y, res.xi, res.theta, res.c_eta = _p(y), _p(xi), _p(theta), _p(c_eta)
    res.history = _p(hist) if record_history else None
    t0 = None if theta0 is None else _c(theta0)
    inner_it = C.c_int64(0)
    rc = lib().cro_papg_k(_p(X), _p(ys), N, n, K, C.byref(cfg), C.byref(icfg), _p(_c(feas_y)),
                          _p(_c(feas_xi).reshape(-1)), _p(t0), C.byref(res), C.byref(inner_it))
    if rc == -4:
        raise RuntimeError("papg: non-finite dual gradient")
    if rc != 0:
        raise RuntimeError(f"oracle papg_k failed ({rc})")
    out = OracleResult(y, xi.reshape(N, n), theta, c_eta, hist[: res.iters], int(res.iters),
                       REASONS[res.reason], res.restarts, bool(res.saturated), res.g_final,
                       res.delta_estimate, res.sigma_C, res.L_g, res.B_theta, res.wall_seconds,
                       res.sigma_iters)
    out.extra["inner_iters"] = inner_it.value
    return out

"""ctypes wrapper for the REFERENCE's own compiled code -- TEST INFRASTRUCTURE ONLY.

Loads oracle/_ref/libcvxreg_ref.so: the reference's proj/core sources compiled
unmodified (oracle/Makefile, target `ref`; Eigen calls served by
oracle/eigen_shim). It exists where /root/reference was present at build time
and travels to the GPU box as a prebuilt file; `available()` says whether it is
there. Same call shapes and result types as oracle/oracle.py, so a test can run
both and compare. Only tests/, scripts/make_ref_golden.py and bench.py's CPU
reference legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import oracle as O
from .oracle import (AlccResult, CroAlccConfig, CroAlccResult, CroConfig, CroResult,
                     INNER_DEFAULTS, OracleResult, Prepared, REASONS, _c, _p, _P)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libcvxreg_ref.so")
# the same sources over the Eigen stand-in's left-to-right reductions (see eigen_shim/Eigen/Dense)
LIB_PATH_SEQ = os.path.join(HERE, "_ref", "libcvxreg_ref_seq.so")
REF_KINDS = {"quadratic": 0, "exponential": 1, "affine-noiseless": 2, "custom-1d": 3}

_lib = None
_lib_seq = None


def build():
    """Compiles oracle/_ref from /root/reference when that tree exists (no-op otherwise)."""
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def available_sequential() -> bool:
    return os.path.exists(LIB_PATH_SEQ)


def lib_sequential():
    """The build with left-to-right reductions; only papg and sigma are bound on it."""
    global _lib_seq
    if _lib_seq is None:
        if not available_sequential():
            raise FileNotFoundError("oracle/_ref/libcvxreg_ref_seq.so absent")
        L = C.CDLL(LIB_PATH_SEQ)
        d, i64, i32 = C.c_double, C.c_int64, C.c_int
        L.ref_last_error.restype = C.c_char_p
        L.ref_sigma.argtypes = [_P, i64, i64, i64, i32, d, i32, _P, C.POINTER(i32), C.POINTER(i32)]
        L.ref_papg.argtypes = [_P, _P, i64, i64, i64, C.POINTER(CroConfig),
                               C.POINTER(CroAlccConfig), i32, _P, _P, _P, C.POINTER(CroResult)]
        _lib_seq = L
    return _lib_seq


def lib():
    global _lib
    if _lib is None:
        if not available():
            build()
        if not available():
            raise FileNotFoundError("oracle/_ref/libcvxreg_ref.so absent (reference tree not "
                                    "present at build time)")
        L = C.CDLL(LIB_PATH)
        d, i64, i32, u64 = C.c_double, C.c_int64, C.c_int, C.c_uint64
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_draws.argtypes = [u64, u64, i64, i32, _P]
        L.ref_gen_instance.argtypes = [i32, i64, i64, d, u64, _P, _P]
        L.ref_validate.argtypes = [_P, _P, i64, i64]
        L.ref_prepare.argtypes = [_P, _P, i64, i64, d, _P, _P, _P, _P, _P, _P, _P]
        L.ref_apply_C.argtypes = [_P, i64, i64, i64, _P, _P, _P]
        L.ref_apply_C_T.argtypes = [_P, i64, i64, i64, _P, _P, _P]
        L.ref_apply_rows.argtypes = [_P, i64, i64, _P, _P, _P]
        L.ref_rows_adjoint.argtypes = [_P, i64, i64, _P, _P, _P]
        L.ref_sigma.argtypes = [_P, i64, i64, i64, i32, d, i32, _P, C.POINTER(i32), C.POINTER(i32)]
        L.ref_cross_position.argtypes = [i64, i64, i64, i64]
        L.ref_cross_position.restype = i64
        L.ref_project_nonneg_ball.argtypes = [_P, i64, d]
        L.ref_project_nonneg_ball.restype = None
        L.ref_momentum_next.argtypes = [d]
        L.ref_momentum_next.restype = d
        L.ref_certificate.argtypes = [d, d, d, d, _P]
        L.ref_certificate.restype = None
        L.ref_papg.argtypes = [_P, _P, i64, i64, i64, C.POINTER(CroConfig),
                               C.POINTER(CroAlccConfig), i32, _P, _P, _P, C.POINTER(CroResult)]
        L.ref_dual_gradient.argtypes = [_P, _P, i64, i64, i64, C.POINTER(CroConfig),
                                        C.POINTER(CroAlccConfig), _P, _P, _P, d, _P, _P, _P, _P]
        L.ref_alcc.argtypes = [_P, _P, i64, i64, d, d, d, _P, _P, C.POINTER(CroAlccConfig),
                               C.POINTER(CroAlccResult)]
        L.ref_infeasibility.argtypes = [_P, i64, i64, _P, _P, _P]
        L.ref_duality_gap.argtypes = [_P, i64, i64, _P, _P, _P, _P]
        L.ref_evaluate_estimator.argtypes = [_P, i64, i64, _P, _P, _P]
        L.ref_evaluate_estimator.restype = d
        L.ref_repair_feasibility.argtypes = [_P, i64, i64, _P, _P, _P]
        _lib = L
    return _lib


def _check(rc, what):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == -1:
        raise ValueError(msg)  # std::invalid_argument
    if rc == -2:
        raise MemoryError(msg)
    raise RuntimeError(f"{what}: {msg}")  # std::runtime_error and the rest


def rng_draws(seed, tag, count, kind="uniform"):
    out = np.empty(count)
    lib().ref_rng_draws(seed, tag, count, {"uniform": 0, "normal": 1}[kind], _p(out))
    return out


def gen_instance(kind, N, n, noise=1.0, seed=1):
    """testgen.cpp gen_instance (the reference's four kinds only)."""
    X = np.empty((N, n))
    y = np.empty(N)
    _check(lib().ref_gen_instance(REF_KINDS[kind], N, n, noise, seed, _p(X), _p(y)), "gen_instance")
    return X, y


def validate(X, y):
    X = _c(X)
    _check(lib().ref_validate(_p(X), _p(_c(y)), X.shape[0], X.shape[1]), "validate_dataset")


def prepare(X, y, gamma=1e-3):
    X = _c(X)
    y = _c(y)
    N, n = X.shape
    ys, shift, fy, fxi = np.empty(N), np.zeros(1), np.empty(N), np.empty(N * n)
    b4, ic, sl = np.empty(4), np.zeros(1), np.empty(n)
    _check(lib().ref_prepare(_p(X), _p(y), N, n, gamma, _p(ys), _p(shift), _p(fy), _p(fxi),
                             _p(b4), _p(ic), _p(sl)), "prepare_problem")
    return Prepared(X, ys, float(shift[0]), fy, fxi, b4[0], b4[1], b4[2], b4[3], float(ic[0]), sl)


def apply_C(X, y, xi, K=None):
    X = _c(X)
    N, n = X.shape
    K = N if K is None else K
    out = np.empty(N * (N - N // K) + N)
    _check(lib().ref_apply_C(_p(X), N, n, K, _p(_c(y)), _p(_c(xi).reshape(-1)), _p(out)), "apply_C")
    return out


def apply_C_T(X, theta, K=None):
    X = _c(X)
    N, n = X.shape
    K = N if K is None else K
    oy, oxi = np.empty(N), np.empty(N * n)
    _check(lib().ref_apply_C_T(_p(X), N, n, K, _p(_c(theta)), _p(oy), _p(oxi)), "apply_C_T")
    return oy, oxi


def apply_rows(X, y, xi):
    X = _c(X)
    N, n = X.shape
    out = np.empty(N * (N - 1))
    _check(lib().ref_apply_rows(_p(X), N, n, _p(_c(y)), _p(_c(xi).reshape(-1)), _p(out)),
           "apply_rows")
    return out


def rows_adjoint(X, z):
    X = _c(X)
    N, n = X.shape
    oy, oxi = np.empty(N), np.empty(N * n)
    _check(lib().ref_rows_adjoint(_p(X), N, n, _p(_c(z)), _p(oy), _p(oxi)), "rows_adjoint")
    return oy, oxi


def sigma(X, which="C", K=None, tol=1e-6, max_iters=5000):
    """estimate_sigma_max on op_C (K blocks; default singleton), op_A1 or op_A2."""
    X = _c(X)
    N, n = X.shape
    s, it, cv = np.zeros(1), C.c_int(0), C.c_int(0)
    _check(lib().ref_sigma(_p(X), N, n, N if K is None else K, {"C": 0, "A1": 1, "A2": 2}[which],
                           tol, max_iters, _p(s), C.byref(it), C.byref(cv)), "estimate_sigma_max")
    return float(s[0]), it.value, bool(cv.value)


def cross_position(N, K, l1, l2):
    r = lib().ref_cross_position(N, K, l1, l2)
    if r < 0:
        raise ValueError("not a cross-block pair")
    return r


def project_nonneg_ball(v, radius):
    v = np.array(v, np.float64)
    lib().ref_project_nonneg_ball(_p(v), v.size, radius)
    return v


def momentum_next(t):
    return lib().ref_momentum_next(t)


def certificate(gamma, delta, B_xi, sigma_):
    out = np.empty(2)
    lib().ref_certificate(gamma, delta, B_xi, sigma_, _p(out))
    return float(out[0]), float(out[1])


def _inner_cfg(inner, threads=1):
    ic = dict(INNER_DEFAULTS)
    ic.update(inner or {})
    return CroAlccConfig(ic["mu1"], ic["tau1_scale"], ic["alpha1_scale"], ic["c"], ic["kappa"],
                         ic["max_outer"], ic["mapg_cap"], ic["infeas_norm_tol"],
                         ic["gap_norm_tol"], ic["max_seconds"], int(ic["record_history"]), threads)


def papg(X, ys, *, K=None, shifted=True, feas_y=None, feas_xi=None, inner=None, gamma=1e-3,
         B_theta=0.0, adaptive_B_theta=True, max_restarts=6, gap_norm_tol=1e-6,
         infeas_norm_tol=1e-1, max_iters=100000, max_seconds=7200.0, inner_tol_floor=1e-6,
         final_resolve_tol=1e-10, record_history=True, use_momentum=True, threads=1,
         theta0=None, want_theta=True, want_c_eta=False, sequential=False):
    """The reference's papg_solve / dual_gradient_ascent (papg.cpp:287-296) with K blocks
    (default K = N: singleton blocks). `shifted=True`: ys are the shifted observations and
    (feas_y, feas_xi) the feasible point of prepare_problem (defaults: prepare() of (X, ys)
    is NOT applied; zeros are used, which only seed the block warm starts and ball radii).
    `shifted=False`: raw ys, prepare_problem runs inside. sigma_C is always the reference's
    own estimate (returned in the result)."""
    X = _c(X)
    ys = _c(ys)
    N, n = X.shape
    K = N if K is None else K
    dim = N * (N - N // K) + N
    cfg = CroConfig(gamma, B_theta, int(adaptive_B_theta), max_restarts, gap_norm_tol,
                    infeas_norm_tol, max_iters, max_seconds, inner_tol_floor, final_resolve_tol,
                    int(record_history), int(use_momentum), 0.0, threads, 0)
    icfg = _inner_cfg(inner)
    y, xi = np.empty(N), np.empty(N * n)
    theta = np.empty(dim) if want_theta else None
    c_eta = np.empty(dim) if want_c_eta else None
    hist = np.zeros((max_iters if record_history else 0, 8))
    res = CroResult()
    res.y, res.xi, res.theta, res.c_eta = _p(y), _p(xi), _p(theta), _p(c_eta)
    res.history = _p(hist) if record_history else None
    fy = _c(feas_y) if feas_y is not None else np.zeros(N)
    fxi = _c(feas_xi).reshape(-1) if feas_xi is not None else np.zeros(N * n)
    t0 = None if theta0 is None else _c(theta0)
    L = lib_sequential() if sequential else lib()
    rc = L.ref_papg(_p(X), _p(ys), N, n, K, C.byref(cfg), C.byref(icfg), int(shifted),
                    _p(fy), _p(fxi), _p(t0), C.byref(res))
    if rc != 0 and sequential:
        raise RuntimeError(f"papg (sequential build): {L.ref_last_error().decode()}")
    _check(rc, "papg")
    return OracleResult(y, xi.reshape(N, n), theta, c_eta, hist[: res.iters], int(res.iters),
                        REASONS[res.reason], res.restarts, bool(res.saturated), res.g_final,
                        res.delta_estimate, res.sigma_C, res.L_g, res.B_theta, res.wall_seconds)


def dual_gradient(X, ys, theta, *, K=None, feas_y=None, feas_xi=None, inner=None, gamma=1e-3,
                  inner_tol=1e-6, threads=1):
    """DualDecomposition::dual_gradient (papg.cpp:89-132) -> (y, xi, C_eta, g, within_infeas,
    inner_iters)."""
    X = _c(X)
    ys = _c(ys)
    N, n = X.shape
    K = N if K is None else K
    dim = N * (N - N // K) + N
    cfg = CroConfig(gamma, 0.0, 1, 6, 1e-6, 1e-1, 1, 7200.0, 1e-6, 1e-10, 1, 1, 0.0, threads, 0)
    icfg = _inner_cfg(inner)
    y, xi, ce, sc = np.empty(N), np.empty(N * n), np.empty(dim), np.empty(3)
    fy = _c(feas_y) if feas_y is not None else np.zeros(N)
    fxi = _c(feas_xi).reshape(-1) if feas_xi is not None else np.zeros(N * n)
    rc = lib().ref_dual_gradient(_p(X), _p(ys), N, n, K, C.byref(cfg), C.byref(icfg), _p(fy),
                                 _p(fxi), _p(_c(theta)), inner_tol, _p(y), _p(xi), _p(ce), _p(sc))
    _check(rc, "dual_gradient")
    return y, xi.reshape(N, n), ce, float(sc[0]), float(sc[1]), int(sc[2])


def alcc(X, ys, *, gamma, Bbar_y, Bbar_xi, warm_y, warm_xi, want_multiplier=False, **inner):
    """The reference's alcc_solve (alcc.cpp:193-208), through the forwarding overload of
    oracle/ref_build/alcc_tu.cpp."""
    X = _c(X)
    ys = _c(ys)
    N, n = X.shape
    threads = inner.pop("threads", 1)
    cfg = _inner_cfg(inner, threads)
    y, xi = np.empty(N), np.empty(N * n)
    mult = np.empty(N * (N - 1)) if want_multiplier else None
    hist = np.zeros((cfg.max_outer, 8))
    res = CroAlccResult()
    res.y, res.xi, res.multiplier, res.history = _p(y), _p(xi), _p(mult), _p(hist)
    res.mapg_iters = None
    rc = lib().ref_alcc(_p(X), _p(ys), N, n, gamma, Bbar_y, Bbar_xi, _p(_c(warm_y)),
                        _p(_c(warm_xi).reshape(-1)), C.byref(cfg), C.byref(res))
    _check(rc, "alcc")
    k = int(res.outer_iters)
    return AlccResult(y, xi.reshape(N, n), mult, hist[:k], np.zeros(0, np.int64), k,
                      int(res.mapg_iters_total), REASONS[res.reason], False, res.certified_gap,
                      res.infeas_raw, res.gap_raw, res.objective, res.wall_seconds, 0.0, 0.0)


def infeasibility(X, y, xi):
    X = _c(X)
    out = np.empty(2)
    _check(lib().ref_infeasibility(_p(X), X.shape[0], X.shape[1], _p(_c(y)),
                                   _p(_c(xi).reshape(-1)), _p(out)), "infeasibility")
    return float(out[0]), float(out[1])


def duality_gap(X, theta, y, xi):
    X = _c(X)
    out = np.empty(2)
    _check(lib().ref_duality_gap(_p(X), X.shape[0], X.shape[1], _p(_c(theta)), _p(_c(y)),
                                 _p(_c(xi).reshape(-1)), _p(out)), "duality_gap")
    return float(out[0]), float(out[1])


def evaluate_estimator(X, y, xi, xq):
    X = _c(X)
    return lib().ref_evaluate_estimator(_p(X), X.shape[0], X.shape[1], _p(_c(y)),
                                        _p(_c(xi).reshape(-1)), _p(_c(xq)))


def repair_feasibility(X, y, xi):
    X = _c(X)
    out = np.empty(X.shape[0])
    _check(lib().ref_repair_feasibility(_p(X), X.shape[0], X.shape[1], _p(_c(y)),
                                        _p(_c(xi).reshape(-1)), _p(out)), "repair_feasibility")
    return out


__all__ = [n for n in dir() if not n.startswith("_")] + ["O"]

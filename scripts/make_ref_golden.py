"""Generates tests/golden/ref_*.npz from the REFERENCE's own compiled code.

oracle/_ref/libcvxreg_ref.so is the reference's proj/core sources compiled
unmodified in this container (oracle/Makefile target `ref`, Eigen calls served
by oracle/eigen_shim); this script runs it through oracle/ref.py and stores
small seeded input/output vectors. The fixtures travel (the reference tree
does not), so the CPU tests pin the oracle restatement to them and the GPU
tests compare the CUDA path with them directly.

    make -C oracle ref && python scripts/make_ref_golden.py

Singleton blocks (the hot path): the reference runs them through
Partition{N, 1} built directly (see oracle/ref_build/ref_capi.cpp). The
per-pair residuals C eta of the k-th iteration are not part of PapgResult;
they are taken from the reference's dual_gradient (papg.cpp:89-132) at
theta2_k, which is rebuilt from the reference's own theta1 after k-1 and k-2
iterations by the extrapolation of papg.cpp:256-262.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (BASELINE generator kinds only: inputs)
from oracle import ref as R  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

# source, kind, N, n, noise, seed, pieces, iters, gap_tol, infeas_tol, B_theta, momentum
SINGLETON = [
    ("oracle-gen", "sqnorm-uniform", 60, 5, 0.1, 1, 0, 40, -1.0, -1.0, 0.0, 1),
    ("oracle-gen", "maxaffine-uniform", 48, 10, 0.1, 2, 20, 30, -1.0, -1.0, 0.0, 1),
    ("oracle-gen", "lse-uniform", 40, 20, 0.05, 3, 50, 25, -1.0, -1.0, 0.0, 1),
    ("oracle-gen", "maxaffine-uniform", 33, 3, 0.1, 4, 5, 35, -1.0, -1.0, 3e-4, 1),  # ball binding
    ("oracle-gen", "sqnorm-uniform", 50, 2, 0.2, 5, 0, 30, -1.0, -1.0, 0.0, 0),      # DGA
    ("oracle-gen", "sqnorm-uniform", 80, 5, 0.1, 6, 0, 5000, 1e-6, 1e-1, 0.0, 1),    # to tolerance
    ("ref-gen", "quadratic", 64, 4, 0.5, 7, 0, 30, -1.0, -1.0, 0.0, 1),              # testgen.cpp
    ("ref-gen", "exponential", 45, 3, 0.2, 8, 0, 30, -1.0, -1.0, 0.0, 1),
    ("ref-gen", "custom-1d", 37, 1, 0.3, 9, 0, 60, -1.0, -1.0, 0.0, 1),
    ("oracle-gen", "maxaffine-uniform", 150, 10, 0.1, 11, 20, 5000, 1e-4, 1e-1, 0.0, 1),  # cfg 2 rule
    # tiny ball + loose thresholds: saturated stops double B_theta (papg.cpp:238-251)
    ("oracle-gen", "sqnorm-uniform", 70, 3, 0.1, 5, 0, 400, 1e9, 1e9, 1e-5, 1),
]
WARM_CASE = 1  # this case is also run from a clipped warm start theta0 (papg.cpp:158-164)

# kind, N, n, K, noise, seed, pieces, iters, inner
GENERAL = [
    ("quadratic", 48, 3, 4, 0.3, 2, 0, 12, dict(max_outer=8, mapg_cap=1500)),
    ("maxaffine-uniform", 60, 4, 5, 0.3, 3, 6, 12, dict(max_outer=8, mapg_cap=1500)),
    ("sqnorm-uniform", 40, 2, 2, 0.3, 4, 0, 10, dict(max_outer=8, mapg_cap=1500)),
]

# kind, N, n, noise, seed, max_outer, mapg_cap
ALCC = [
    ("quadratic", 40, 3, 0.5, 9, 6, 2000),
    ("exponential", 36, 2, 0.2, 10, 5, 1500),
]


def momentum_beta(k):
    """(t_{k-1} - 1) / t_k of engines.hpp:11-13 from t_1 = 1: the coefficient that builds
    theta2_k after iteration k-1 (papg.cpp:256-262)."""
    t = 1.0
    for _ in range(k - 2):
        t = R.momentum_next(t)
    return (t - 1.0) / R.momentum_next(t)


def data_for(source, kind, N, n, noise, seed, pieces):
    if source == "ref-gen":
        return R.gen_instance(kind, N, n, noise, seed)
    return O.gen_instance(kind, N, n, noise, seed, pieces)


def singleton():
    d = {"count": np.array(len(SINGLETON))}
    for i, (src, kind, N, n, noise, seed, pieces, iters, gt, ft, B, mom) in enumerate(SINGLETON):
        X, y = data_for(src, kind, N, n, noise, seed, pieces)
        P = R.prepare(X, y)
        kw = dict(feas_y=P.feas_y, feas_xi=P.feas_xi, gap_norm_tol=gt, infeas_norm_tol=ft,
                  B_theta=B, use_momentum=bool(mom))
        r = R.papg(X, P.ys, max_iters=iters, **kw)
        k = r.iters
        c_eta = np.zeros(0)
        if r.restarts == 0 and k >= 3:
            kwf = dict(kw, gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
            a = R.papg(X, P.ys, max_iters=k - 1, **kwf).theta
            if mom:
                b = R.papg(X, P.ys, max_iters=k - 2, **kwf).theta
                theta2 = a + momentum_beta(k) * (a - b)
            else:
                theta2 = a
            c_eta = R.dual_gradient(X, P.ys, theta2, feas_y=P.feas_y, feas_xi=P.feas_xi)[2]
        d[f"X{i}"] = X
        d[f"yraw{i}"] = y
        d[f"ys{i}"] = P.ys
        d[f"feas{i}"] = np.concatenate([P.feas_y, P.feas_xi])
        d[f"meta{i}"] = np.array([iters, r.sigma_C, gt, ft, B, mom], np.float64)
        d[f"theta{i}"] = r.theta
        d[f"c_eta{i}"] = c_eta
        d[f"y{i}"] = r.y
        d[f"xi{i}"] = r.xi
        d[f"hist{i}"] = r.history[:, :7]
        d[f"iters{i}"] = np.array([r.iters, r.restarts, O.REASONS_INV[r.reason], int(r.saturated)])
        d[f"scal{i}"] = np.array([r.g_final, r.delta_estimate, r.B_theta, r.L_g])
        sg = R.sigma(X)
        d[f"sigma{i}"] = np.array([sg[0], sg[1], int(sg[2])], np.float64)
        if i == WARM_CASE:
            theta0 = r.theta * 3e4 + np.random.default_rng(0).normal(size=r.theta.size) * 1e-3
            w = R.papg(X, P.ys, max_iters=20, theta0=theta0, **dict(kw, B_theta=20.0))
            d["warm_theta0"] = theta0
            d["warm_theta"] = w.theta
            d["warm_y"] = w.y
            d["warm_hist"] = w.history[:, :7]
        print("singleton", src, kind, N, n, "iters", r.iters, r.reason, "restarts", r.restarts,
              "c_eta", c_eta.size > 0)
    np.savez_compressed(os.path.join(OUT, "ref_papg_singleton.npz"), **d)


def general():
    d = {"count": np.array(len(GENERAL))}
    for i, (kind, N, n, K, noise, seed, pieces, iters, inner) in enumerate(GENERAL):
        X, y = O.gen_instance(kind, N, n, noise, seed, pieces)
        P = R.prepare(X, y)
        r = R.papg(X, P.ys, K=K, feas_y=P.feas_y, feas_xi=P.feas_xi, inner=inner, max_iters=iters,
                   gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
        d[f"X{i}"] = X
        d[f"ys{i}"] = P.ys
        d[f"feas{i}"] = np.concatenate([P.feas_y, P.feas_xi])
        d[f"meta{i}"] = np.array([iters, r.sigma_C, K, inner["max_outer"], inner["mapg_cap"]],
                                 np.float64)
        d[f"theta{i}"] = r.theta
        d[f"y{i}"] = r.y
        d[f"xi{i}"] = r.xi
        d[f"hist{i}"] = r.history[:, :7]
        d[f"scal{i}"] = np.array([r.g_final, r.delta_estimate, r.B_theta, r.L_g])
        sg = R.sigma(X, "C", K)
        d[f"sigma{i}"] = np.array([sg[0], sg[1], int(sg[2])], np.float64)
        print("general", kind, N, n, K, "iters", r.iters, r.reason)
    np.savez_compressed(os.path.join(OUT, "ref_papg_general.npz"), **d)


def alcc():
    d = {"count": np.array(len(ALCC))}
    for i, (kind, N, n, noise, seed, max_outer, cap) in enumerate(ALCC):
        X, y = R.gen_instance(kind, N, n, noise, seed)
        P = R.prepare(X, y)
        s1, s2 = R.sigma(X, "A1"), R.sigma(X, "A2")
        a = R.alcc(X, P.ys, gamma=1e-3, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, warm_y=P.feas_y,
                   warm_xi=P.feas_xi, max_outer=max_outer, mapg_cap=cap, want_multiplier=True)
        d[f"X{i}"] = X
        d[f"ys{i}"] = P.ys
        d[f"feas{i}"] = np.concatenate([P.feas_y, P.feas_xi])
        d[f"meta{i}"] = np.array([max_outer, cap, P.Bbar_y, P.Bbar_xi, s1[0], s2[0], s1[1], s2[1]])
        d[f"y{i}"] = a.y
        d[f"xi{i}"] = a.xi
        d[f"mult{i}"] = a.multiplier
        d[f"hist{i}"] = a.history[:, :7]
        d[f"scal{i}"] = np.array([a.outer_iters, a.mapg_iters_total, O.REASONS_INV[a.reason],
                                  a.certified_gap, a.infeas_raw, a.gap_raw, a.objective])
        print("alcc", kind, N, n, "outer", a.outer_iters, "mapg", a.mapg_iters_total, a.reason)
    np.savez_compressed(os.path.join(OUT, "ref_alcc.npz"), **d)


def operators():
    rng = np.random.default_rng(12)
    X, y = R.gen_instance("quadratic", 30, 3, 0.4, 21)
    N, n = X.shape
    P = R.prepare(X, y)
    yy, xi = rng.standard_normal(N), rng.standard_normal((N, n))
    d = dict(X=X, yraw=y, yy=yy, xi=xi, ys=P.ys, feas=np.concatenate([P.feas_y, P.feas_xi]),
             prep=np.array([P.shift, P.B_theta, P.Bbar_y, P.Bbar_xi, P.intercept]), slope=P.slope)
    for K in (N, 5, 2):
        th = rng.random(N * (N - N // K) + N)
        d[f"theta_K{K}"] = th
        d[f"C_K{K}"] = R.apply_C(X, yy, xi, K)
        oy, oxi = R.apply_C_T(X, th, K)
        d[f"CT_K{K}"] = np.concatenate([oy, oxi])
        sg = R.sigma(X, "C", K)
        d[f"sigma_K{K}"] = np.array([sg[0], sg[1], int(sg[2])], np.float64)
    z = rng.random(N * (N - 1))
    d["z"] = z
    d["rows"] = R.apply_rows(X, yy, xi)
    oy, oxi = R.rows_adjoint(X, z)
    d["rows_adj"] = np.concatenate([oy, oxi])
    d["sigma_A"] = np.array([*R.sigma(X, "A1")[:2], *R.sigma(X, "A2")[:2]], np.float64)
    th = d[f"theta_K{N}"]
    d["metrics"] = np.array([*R.infeasibility(X, yy, xi), *R.duality_gap(X, th, yy, xi),
                             R.evaluate_estimator(X, yy, xi, X[3] + 0.1)])
    d["repair"] = R.repair_feasibility(X, yy, xi)
    v = rng.standard_normal(50)
    d["proj_in"] = v
    d["proj_out"] = R.project_nonneg_ball(v, 2.0)
    t, ts = 1.0, []
    for _ in range(8):
        t = R.momentum_next(t)
        ts.append(t)
    d["momentum"] = np.array(ts)
    d["certificate"] = np.array(R.certificate(1e-3, 0.02, 3.0, 40.0))
    for kind, nn in (("quadratic", 3), ("exponential", 4), ("affine-noiseless", 2), ("custom-1d", 1)):
        Xg, yg = R.gen_instance(kind, 25, nn, 0.3, 5)
        d[f"gen_{kind}"] = np.concatenate([Xg.reshape(-1), yg])
    d["rng_uniform_7_3"] = R.rng_draws(7, 3, 16, "uniform")
    d["rng_normal_5eed_97"] = R.rng_draws(0x5EED, 97, 16, "normal")
    np.savez_compressed(os.path.join(OUT, "ref_operators.npz"), **d)
    print("operators ok")


if __name__ == "__main__":
    if not R.available():
        R.build()
    os.makedirs(OUT, exist_ok=True)
    singleton()
    general()
    alcc()
    operators()

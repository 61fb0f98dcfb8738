"""Pins the CPU oracle (oracle/cvxreg_oracle.c) before it is trusted.

The reference ships no tests or golden vectors for this path (SURVEY.md
section 4, 8c), so the oracle is pinned against
  * the SPEC.md worked examples of the operations on the path,
  * analytic known-answer tests,
  * an independent dense numpy restatement (explicit C matrix) of the same
    loop, papg.cpp:136-283, on tiny instances,
  * the committed golden fixtures (tests/golden, made by scripts/make_golden.py).
"""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- SPEC examples
def test_projection_examples(oracle):  # SPEC.md:193-195 (projections.hpp:9-13)
    assert np.allclose(oracle.project_nonneg_ball([-1.0, 3.0, 4.0], 5.0), [0.0, 3.0, 4.0])
    assert np.allclose(oracle.project_nonneg_ball([3.0, 4.0], 1.0), [0.6, 0.8])
    rng = np.random.default_rng(0)
    v = rng.normal(size=50) * 3
    p1 = oracle.project_nonneg_ball(v, 2.0)
    assert np.allclose(oracle.project_nonneg_ball(p1, 2.0), p1)  # idempotence
    assert (p1 >= 0).all() and np.linalg.norm(p1) <= 2.0 + 1e-12


def test_momentum_sequence(oracle):  # SPEC.md:213 (engines.hpp:11-13)
    t2 = oracle.momentum_next(1.0)
    t3 = oracle.momentum_next(t2)
    # SPEC.md:213 quotes t3 ~ 2.1754, which its own rule contradicts:
    # (1 + sqrt(1 + 4 * 1.6180^2)) / 2 = 2.1935. engines.hpp:11-13 is followed.
    assert abs(t2 - 1.6180) < 1e-4 and abs(t3 - 2.1935) < 1e-4
    t = 1.0
    for ell in range(1, 200):  # t_l >= (l+1)/2
        assert t >= (ell + 1) / 2 - 1e-12
        t = oracle.momentum_next(t)


def test_cross_position(oracle):  # SPEC.md:60-62 (indexing.hpp:30-37), 0-based
    assert oracle.cross_position(4, 2, 0, 2) == 0
    assert oracle.cross_position(4, 2, 3, 1) == 7
    with pytest.raises(ValueError):
        oracle.cross_position(4, 2, 0, 1)
    # singleton partition: cross order == full lexicographic order, diagonal skipped
    N = 7
    r = 0
    for l1 in range(N):
        for l2 in range(N):
            if l1 != l2:
                assert oracle.cross_position(N, N, l1, l2) == r
                r += 1


def test_apply_C_examples(oracle):
    X = np.array([[0.0], [1.0]])
    # within-block example (9, -7): rows (1,2), (2,1) of A1 y + A2 xi
    out = oracle.apply_C(X, np.array([3.0, 1.0]), np.array([5.0, 7.0]))
    assert np.allclose(out[:2], [9.0, -7.0]) and np.allclose(out[2:], [3.0, 1.0])
    # constant y, xi = 0: cross rows vanish, identity rows pass y
    rng = np.random.default_rng(1)
    X = rng.normal(size=(4, 2))
    out = oracle.apply_C(X, np.full(4, 2.5), np.zeros(8))
    assert np.all(out[:12] == 0) and np.all(out[12:] == 2.5)
    # affine y = a + b.x, xi = b: all cross rows are 0
    b = rng.normal(size=2)
    y = 0.7 + X @ b
    out = oracle.apply_C(X, y, np.tile(b, 4))
    assert np.abs(out[:12]).max() < 1e-12


def test_infeasibility_hand_example(oracle):
    X = np.array([[0.0], [1.0]])
    out = oracle.apply_C(X, np.zeros(2), np.array([0.0, -1.0]))
    raw = np.linalg.norm(np.minimum(out[:2], 0))
    assert raw == 1.0 and abs(raw / np.sqrt(2) - 1 / np.sqrt(2)) < 1e-15


def test_adjoint_identity_and_unit_vectors(oracle):
    rng = np.random.default_rng(2)
    N, n = 9, 3
    X = rng.normal(size=(N, n))
    y, xi = rng.normal(size=N), rng.normal(size=N * n)
    th = rng.normal(size=N * (N - 1) + N)
    Ce = oracle.apply_C(X, y, xi)
    oy, oxi = oracle.apply_C_T(X, th)
    lhs, rhs = Ce @ th, y @ oy + xi @ oxi
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1.0)
    # one-hot theta at row (l1, l2): +1 at l1, -1 at l2, -(x_l1 - x_l2) in xi_l2
    l1, l2 = 2, 5
    e = np.zeros_like(th)
    e[oracle.cross_position(N, N, l1, l2)] = 1.0
    oy, oxi = oracle.apply_C_T(X, e)
    ey = np.zeros(N)
    ey[l1], ey[l2] = 1.0, -1.0
    exi = np.zeros((N, n))
    exi[l2] = -(X[l1] - X[l2])
    assert np.allclose(oy, ey) and np.allclose(oxi.reshape(N, n), exi)


def _dense_C(X):
    N, n = X.shape
    rows = []
    for l1 in range(N):
        for l2 in range(N):
            if l1 == l2:
                continue
            r = np.zeros(N + N * n)
            r[l1] += 1.0
            r[l2] -= 1.0
            r[N + l2 * n: N + (l2 + 1) * n] = -(X[l1] - X[l2])
            rows.append(r)
    for l in range(N):
        r = np.zeros(N + N * n)
        r[l] = 1.0
        rows.append(r)
    return np.array(rows)


def test_sigma_C_vs_dense_svd(oracle):
    rng = np.random.default_rng(3)
    for N, n in [(6, 1), (8, 2), (12, 3)]:
        X = rng.normal(size=(N, n))
        smax = np.linalg.svd(_dense_C(X), compute_uv=False)[0]
        s, it, conv = oracle.sigma_C(X)
        assert conv
        assert s / 1.01 >= smax * (1 - 1e-3) and s / 1.01 <= smax * 1.001


def test_certificate_arithmetic(oracle):  # SPEC.md:376-377 (papg.cpp:298-303)
    a, b = oracle.certificate(0.04, 1e-4, 1.0, 2.0)
    assert abs(a - 0.3414) < 1e-4 and abs(b - 0.1414) < 1e-4
    a, b = oracle.certificate(0.04, 0.0, 1.0, 2.0)
    assert a == pytest.approx(0.2) and b == 0.0


def test_prepare_examples(oracle):  # SPEC.md:215-233 (preprocess.cpp)
    rng = np.random.default_rng(4)
    X = rng.normal(size=(10, 2))
    # constant data: a = c, b = 0, feasibility residual 0
    p = oracle.prepare(X, np.full(10, 3.0), 1e-3)
    assert abs(p.intercept - 3.0) < 1e-12 and np.abs(p.slope).max() < 1e-12
    # exact affine data: Bbar floored at 1e-8, shift = max(0, Bbar - min y)
    y = 1.0 + X @ np.array([0.5, -2.0])
    p = oracle.prepare(X, y, 1e-3)
    assert p.Bbar_y == pytest.approx(max(np.sqrt(1e-3 * 10 * (0.25 + 4.0)), 1e-8))
    assert p.shift == pytest.approx(max(0.0, p.Bbar_y - y.min()))
    assert np.allclose(p.ys, y + p.shift)
    # affine feasible point satisfies every row with equality
    Ce = oracle.apply_C(X, p.feas_y, p.feas_xi)
    assert np.abs(Ce[:90]).max() < 1e-12


# ------------------------------------------------------------ known answers
def test_first_iterate_known_answer(oracle):
    X, y = oracle.gen_instance("sqnorm-uniform", 40, 3, 0.1, 5)
    p = oracle.prepare(X, y)
    s, _, _ = oracle.sigma_C(X)
    L = s * s / 1e-3
    r = oracle.papg(X, p.ys, max_iters=1, sigma_C=s, gap_norm_tol=-1, infeas_norm_tol=-1,
                    want_c_eta=True)
    N = 40
    ys = p.ys
    exp = np.array([max(ys[l2] - ys[l1], 0.0) / L for l1 in range(N) for l2 in range(N) if l1 != l2])
    assert np.linalg.norm(exp) <= r.B_theta  # ball not binding
    assert np.allclose(r.theta[: N * (N - 1)], exp, rtol=1e-12, atol=1e-300)
    assert np.all(r.theta[N * (N - 1):] == 0.0)  # shifted ybar > 0
    rows = np.array([ys[l1] - ys[l2] for l1 in range(N) for l2 in range(N) if l1 != l2])
    assert np.allclose(r.c_eta[: N * (N - 1)], rows, rtol=1e-14)
    gap = -np.sum(np.maximum(-rows, 0) ** 2) / L
    assert r.history[0, 5] == pytest.approx(gap, rel=1e-12)


def test_diagonal_free_and_feasible_set(oracle):  # A.4.3, theta in Q2 (papg invariants)
    X, y = oracle.gen_instance("maxaffine-uniform", 30, 2, 0.1, 2, 4)
    p = oracle.prepare(X, y)
    r = oracle.papg(X, p.ys, max_iters=50, gap_norm_tol=-1, infeas_norm_tol=-1, B_theta=1e-3,
                    adaptive_B_theta=False)
    assert r.theta.min() >= 0.0
    assert np.linalg.norm(r.theta) <= 1e-3 * (1 + 1e-12)


# ------------------------------------------------------- dense restatement
def _dense_papg(X, ys, sigma, gamma, iters, B, momentum=True):
    """papg.cpp:136-283 with an explicit C matrix (numpy), singleton blocks."""
    N, n = X.shape
    C = _dense_C(X)
    L = sigma * sigma / gamma
    th1 = np.zeros(C.shape[0])
    th1p = th1.copy()
    th2 = th1.copy()
    t = 1.0
    hist = []
    for ell in range(1, iters + 1):
        q = C.T @ th2
        y = ys + q[:N]
        xi = q[N:] / gamma
        Ce = C @ np.concatenate([y, xi])
        th1p, th1 = th1, np.maximum(th2 - Ce / L, 0)
        nrm = np.linalg.norm(th1)
        if nrm > B:
            th1 = th1 * (B / nrm)
        hist.append(((th1 if momentum else th2) @ Ce, np.linalg.norm(np.minimum(Ce[:-N], 0))))
        if momentum:
            tn = 0.5 * (1 + np.sqrt(1 + 4 * t * t))
            th2 = th1 + ((t - 1) / tn) * (th1 - th1p)
            t = tn
        else:
            th2 = th1.copy()
    q = C.T @ th1
    return th1, ys + q[:N], q[N:] / gamma, np.array(hist)


@pytest.mark.parametrize("momentum", [True, False])
@pytest.mark.parametrize("B", [0.0, 2e-4])
def test_oracle_matches_dense_restatement(oracle, momentum, B):
    X, y = oracle.gen_instance("lse-uniform", 12, 3, 0.05, 9, 5)
    p = oracle.prepare(X, y)
    s, _, _ = oracle.sigma_C(X)
    Bt = B if B > 0 else 10 * np.sqrt(12)
    r = oracle.papg(X, p.ys, max_iters=80, sigma_C=s, gap_norm_tol=-1, infeas_norm_tol=-1,
                    B_theta=B, use_momentum=momentum)
    th, yd, xid, hist = _dense_papg(X, p.ys, s, 1e-3, 80, Bt, momentum)
    assert np.linalg.norm(r.theta - th) <= 1e-12 * np.linalg.norm(th)
    assert np.linalg.norm(r.y - yd) <= 1e-12 * np.linalg.norm(yd)
    assert np.allclose(r.history[:, 5], hist[:, 0], rtol=1e-10, atol=1e-300)
    assert np.allclose(r.history[:, 3], hist[:, 1], rtol=1e-10, atol=1e-300)


def test_openmp_variant_matches_single_thread(oracle):
    X, y = oracle.gen_instance("maxaffine-uniform", 120, 4, 0.1, 3, 6)
    p = oracle.prepare(X, y)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=60, sigma_C=s, gap_norm_tol=-1, infeas_norm_tol=-1)
    a = oracle.papg(X, p.ys, threads=1, **kw)
    b = oracle.papg(X, p.ys, threads=4, **kw)
    assert np.linalg.norm(a.theta - b.theta) <= 1e-12 * np.linalg.norm(a.theta)
    assert np.linalg.norm(a.y - b.y) <= 1e-13 * np.linalg.norm(a.y)


def test_regularised_fit_close_to_qp_solution(oracle):
    """Tiny-instance optimality (SPEC.md:359-360 in spirit): a long P-APG run
    approaches the solution of the regularised QP (Eq. 10) found by SLSQP."""
    scipy = pytest.importorskip("scipy.optimize")
    X, y = oracle.gen_instance("sqnorm-uniform", 6, 1, 0.1, 3)
    p = oracle.prepare(X, y, 1e-2)
    N, n = X.shape
    C = _dense_C(X)[: N * (N - 1)]

    def f(z):
        return 0.5 * np.sum((z[:N] - p.ys) ** 2) + 0.5 * 1e-2 * np.sum(z[N:] ** 2)

    res = scipy.minimize(f, np.concatenate([p.feas_y, p.feas_xi]), jac=lambda z: np.concatenate(
        [z[:N] - p.ys, 1e-2 * z[N:]]), constraints=[{"type": "ineq", "fun": lambda z: C @ z,
                                                       "jac": lambda z: C}],
        method="SLSQP", options={"ftol": 1e-14, "maxiter": 500})
    r = oracle.papg(X, p.ys, gamma=1e-2, max_iters=20000, gap_norm_tol=-1, infeas_norm_tol=-1)
    assert np.abs(r.y - res.x[:N]).max() < 1e-3


# ------------------------------------------------------------------ golden
def test_oracle_reproduces_golden_fixtures(oracle):
    path = os.path.join(GOLDEN, "papg_small.npz")
    g = np.load(path)
    for i in range(int(g["count"])):
        X, ys = g[f"X{i}"], g[f"ys{i}"]
        meta = g[f"meta{i}"]
        r = oracle.papg(X, ys, max_iters=int(meta[0]), sigma_C=float(meta[1]),
                        gap_norm_tol=float(meta[2]), infeas_norm_tol=float(meta[3]),
                        B_theta=float(meta[4]), use_momentum=bool(meta[5]), want_c_eta=True)
        assert r.iters == int(g[f"iters{i}"][0])
        assert np.linalg.norm(r.theta - g[f"theta{i}"]) <= 1e-13 * np.linalg.norm(g[f"theta{i}"])
        assert np.linalg.norm(r.y - g[f"y{i}"]) <= 1e-14 * np.linalg.norm(g[f"y{i}"])


def test_rng_streams_golden(oracle):
    g = np.load(os.path.join(GOLDEN, "rng.npz"))
    assert np.array_equal(oracle.rng_draws(1, 2, 8, "raw53"), g["raw_1_2"])
    assert np.array_equal(oracle.rng_draws(0x5EED, 97, 8, "normal"), g["normal_5eed_97"])
    assert np.array_equal(oracle.rng_draws(7, 3, 8, "uniform"), g["uniform_7_3"])


# ------------------------------------------------------------- metrics.cpp
def test_metrics_examples(oracle):  # SPEC.md:425-440 (metrics.cpp:8-56)
    X = np.array([[0.0], [1.0]])
    raw, norm = oracle.infeasibility(X, np.zeros(2), np.array([0.0, -1.0]))
    assert raw == 1.0 and norm == pytest.approx(1 / np.sqrt(2))
    rng = np.random.default_rng(5)
    X = rng.normal(size=(15, 3))
    b = rng.normal(size=3)
    y = 0.3 + X @ b  # affine point: feasible, estimator reproduces the affine function
    assert oracle.infeasibility(X, y, np.tile(b, 15))[0] < 1e-12
    q = rng.normal(size=3)
    assert oracle.evaluate_estimator(X, y, np.tile(b, 15), q) == pytest.approx(0.3 + q @ b)
    # repair: y'_l = fhat(x_l) >= y_l. metrics.hpp:38 claims (y', xi) is then
    # exactly feasible; that holds only when xi_l is the active slope of fhat at
    # x_l, so we check y' >= y and that it is exact on a consistent point.
    y2, xi2 = rng.normal(size=15), rng.normal(size=45)
    yr = oracle.repair_feasibility(X, y2, xi2)
    assert np.all(yr >= y2 - 1e-12)
    assert np.allclose(oracle.repair_feasibility(X, y, np.tile(b, 15)), y, atol=1e-12)
    # duality gap = theta . C eta (metrics.cpp:17-30)
    th = np.abs(rng.normal(size=15 * 14 + 15))
    g, gn = oracle.duality_gap(X, th, y2, xi2)
    assert g == pytest.approx(th @ oracle.apply_C(X, y2, xi2), rel=1e-12)
    assert gn == pytest.approx(g / (15 * 14))

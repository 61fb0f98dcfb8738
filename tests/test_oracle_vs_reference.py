"""Pins the CPU oracle (oracle/cvxreg_oracle.c) to the REFERENCE's own code.

Two layers:
  * committed fixtures tests/golden/ref_*.npz -- outputs of the reference's
    proj/core sources compiled unmodified in the build container
    (oracle/Makefile target `ref`, scripts/make_ref_golden.py). They always run.
  * live comparisons against oracle/_ref/libcvxreg_ref.so when it is present
    (it is wherever /root/reference existed at build time, and it travels to the
    GPU box as a prebuilt file); skipped otherwise.

Bars: operators, generators, PRNG streams, sigma step counts and the singleton
(K = N) P-APG trajectory are compared BITWISE or to 1e-13 -- the oracle follows
the reference's loop order; only Eigen-side reductions (norm, dot) may differ
in the last bits. The general-K path runs thousands of inner MAPG steps per
block solve: identical iteration counts, iterates within 1e-10.
"""
import os

import numpy as np
import pytest

from oracle import ref as R

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
live = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (no reference tree)")


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def hist_close(h, g, rtol):
    h, g = np.asarray(h)[:, :7], np.asarray(g)[:, :7]
    assert h.shape == g.shape
    assert np.array_equal(h[:, 0], g[:, 0])
    for col in range(1, 7):
        scale = max(np.abs(g[:, col]).max(), 1e-300)
        assert np.abs(h[:, col] - g[:, col]).max() <= rtol * scale, col


# --------------------------------------------------------------- fixtures (always)
def test_oracle_reproduces_reference_singleton_fixtures(oracle):
    g = np.load(os.path.join(GOLDEN, "ref_papg_singleton.npz"))
    assert int(g["count"]) >= 10
    for i in range(int(g["count"])):
        X, ys = g[f"X{i}"], g[f"ys{i}"]
        iters, sigma, gt, ft, B, mom = g[f"meta{i}"]
        want_rows = g[f"c_eta{i}"].size > 0
        r = oracle.papg(X, ys, max_iters=int(iters), sigma_C=float(sigma), gap_norm_tol=float(gt),
                        infeas_norm_tol=float(ft), B_theta=float(B), use_momentum=bool(mom),
                        want_c_eta=True)
        k, restarts, reason, saturated = (int(v) for v in g[f"iters{i}"])
        assert (r.iters, r.restarts, oracle.REASONS_INV[r.reason], int(r.saturated)) == \
            (k, restarts, reason, saturated), i
        assert rel(r.theta, g[f"theta{i}"]) <= 1e-13, (i, rel(r.theta, g[f"theta{i}"]))
        assert rel(r.y, g[f"y{i}"]) <= 1e-13 and rel(r.xi, g[f"xi{i}"]) <= 1e-13
        if want_rows:  # per-pair residuals of the k-th iteration
            assert rel(r.c_eta, g[f"c_eta{i}"]) <= 1e-13, (i, rel(r.c_eta, g[f"c_eta{i}"]))
        hist_close(r.history, g[f"hist{i}"], 1e-11)
        gf, de, Bt, Lg = g[f"scal{i}"]
        assert r.g_final == pytest.approx(gf, rel=1e-12, abs=1e-13)
        assert r.delta_estimate == pytest.approx(de, rel=1e-10, abs=1e-12)
        assert r.B_theta == Bt and r.L_g == pytest.approx(Lg, rel=1e-15)
        # sigma_max(C): the oracle's literal power iteration against the reference's
        s, it, cv = oracle.sigma_C(X)
        assert (it, int(cv)) == (int(g[f"sigma{i}"][1]), int(g[f"sigma{i}"][2]))
        assert s == pytest.approx(g[f"sigma{i}"][0], rel=1e-13)
        # prepare_problem: shifted observations from the raw ones
        P = oracle.prepare(X, g[f"yraw{i}"])
        assert np.abs(P.ys - ys).max() <= 1e-13 * np.abs(ys).max()
        feas = np.concatenate([P.feas_y, P.feas_xi])
        assert rel(feas, g[f"feas{i}"]) <= 1e-12


def test_oracle_reproduces_reference_warm_start_fixture(oracle):
    g = np.load(os.path.join(GOLDEN, "ref_papg_singleton.npz"))
    i = 1
    kw = dict(max_iters=20, sigma_C=float(g[f"meta{i}"][1]), gap_norm_tol=-1.0,
              infeas_norm_tol=-1.0, B_theta=20.0, theta0=g["warm_theta0"])
    r = oracle.papg(g[f"X{i}"], g[f"ys{i}"], **kw)
    assert rel(r.theta, g["warm_theta"]) <= 1e-13 and rel(r.y, g["warm_y"]) <= 1e-13
    hist_close(r.history, g["warm_hist"], 1e-11)


def test_oracle_reproduces_reference_general_k_fixtures(oracle):
    g = np.load(os.path.join(GOLDEN, "ref_papg_general.npz"))
    for i in range(int(g["count"])):
        X, ys, feas = g[f"X{i}"], g[f"ys{i}"], g[f"feas{i}"]
        N, n = X.shape
        iters, sigma, K, mo, cap = g[f"meta{i}"]
        r = oracle.papg_k(X, ys, int(K), feas[:N], feas[N:], inner=dict(max_outer=int(mo),
                          mapg_cap=int(cap)), sigma_C=float(sigma), max_iters=int(iters),
                          gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
        assert r.iters == int(iters)
        assert rel(r.theta, g[f"theta{i}"]) <= 1e-10, rel(r.theta, g[f"theta{i}"])
        assert rel(r.y, g[f"y{i}"]) <= 1e-10 and rel(r.xi, g[f"xi{i}"]) <= 1e-9
        hist_close(r.history, g[f"hist{i}"], 1e-8)
        assert r.g_final == pytest.approx(g[f"scal{i}"][0], rel=1e-10)
        s, it, cv = oracle.sigma_C_k(X, int(K))
        assert (it, int(cv)) == (int(g[f"sigma{i}"][1]), int(g[f"sigma{i}"][2]))
        assert s == pytest.approx(g[f"sigma{i}"][0], rel=1e-13)


def test_oracle_reproduces_reference_alcc_fixtures(oracle):
    g = np.load(os.path.join(GOLDEN, "ref_alcc.npz"))
    for i in range(int(g["count"])):
        X, ys, feas = g[f"X{i}"], g[f"ys{i}"], g[f"feas{i}"]
        N = X.shape[0]
        mo, cap, By, Bxi, s1, s2, it1, it2 = g[f"meta{i}"]
        assert oracle.sigma_A(X, 1)[:2] == (pytest.approx(s1, rel=1e-13), int(it1))
        assert oracle.sigma_A(X, 2)[:2] == (pytest.approx(s2, rel=1e-13), int(it2))
        a = oracle.alcc(X, ys, gamma=1e-3, Bbar_y=By, Bbar_xi=Bxi, warm_y=feas[:N],
                        warm_xi=feas[N:], sigma_A1=s1, sigma_A2=s2, max_outer=int(mo),
                        mapg_cap=int(cap), want_multiplier=True)
        outer, mapg, reason, cert, infeas, gap, obj = g[f"scal{i}"]
        assert (a.outer_iters, a.mapg_iters_total, oracle.REASONS_INV[a.reason]) == \
            (int(outer), int(mapg), int(reason))
        assert rel(a.y, g[f"y{i}"]) <= 1e-12 and rel(a.xi, g[f"xi{i}"]) <= 1e-12
        assert rel(a.multiplier, g[f"mult{i}"]) <= 1e-12
        hist_close(a.history, g[f"hist{i}"], 1e-10)
        assert a.certified_gap == pytest.approx(cert, rel=1e-10)
        assert a.objective == pytest.approx(obj, rel=1e-12)


def test_oracle_reproduces_reference_operator_fixtures(oracle):
    g = np.load(os.path.join(GOLDEN, "ref_operators.npz"))
    X, yy, xi = g["X"], g["yy"], g["xi"]
    N, n = X.shape
    for K in (N, 5, 2):
        th = g[f"theta_K{K}"]
        c = oracle.apply_C(X, yy, xi) if K == N else oracle.apply_C_k(X, K, yy, xi)
        oy, oxi = oracle.apply_C_T(X, th) if K == N else oracle.apply_C_T_k(X, K, th)
        assert np.array_equal(c, g[f"C_K{K}"])  # same loop order: bitwise
        assert np.array_equal(np.concatenate([oy, oxi]), g[f"CT_K{K}"])
        s, it, cv = oracle.sigma_C(X) if K == N else oracle.sigma_C_k(X, K)
        assert (it, int(cv)) == (int(g[f"sigma_K{K}"][1]), int(g[f"sigma_K{K}"][2]))
        assert s == pytest.approx(g[f"sigma_K{K}"][0], rel=1e-13)
    P = oracle.prepare(X, g["yraw"])
    got = np.array([P.shift, P.B_theta, P.Bbar_y, P.Bbar_xi, P.intercept])
    assert np.allclose(got, g["prep"], rtol=1e-12, atol=1e-13)
    assert np.allclose(P.slope, g["slope"], rtol=1e-11, atol=1e-13)
    th = g[f"theta_K{N}"]
    m = np.array([*oracle.infeasibility(X, yy, xi), *oracle.duality_gap(X, th, yy, xi),
                  oracle.evaluate_estimator(X, yy, xi, X[3] + 0.1)])
    assert np.allclose(m, g["metrics"], rtol=1e-13)
    assert np.array_equal(oracle.repair_feasibility(X, yy, xi), g["repair"])
    assert np.allclose(oracle.project_nonneg_ball(g["proj_in"], 2.0), g["proj_out"], rtol=1e-15)
    t, ts = 1.0, []
    for _ in range(8):
        t = oracle.momentum_next(t)
        ts.append(t)
    assert np.array_equal(np.array(ts), g["momentum"])
    assert np.allclose(oracle.certificate(1e-3, 0.02, 3.0, 40.0), g["certificate"], rtol=1e-15)
    for kind, nn in (("quadratic", 3), ("exponential", 4), ("affine-noiseless", 2), ("custom-1d", 1)):
        Xg, yg = oracle.gen_instance(kind, 25, nn, 0.3, 5)
        ref = g[f"gen_{kind}"]
        assert np.array_equal(Xg.reshape(-1), ref[: 25 * nn])  # PRNG + Box-Muller: bitwise
        assert np.allclose(yg, ref[25 * nn:], rtol=1e-13, atol=1e-14)
    assert np.array_equal(oracle.rng_draws(7, 3, 16, "uniform"), g["rng_uniform_7_3"])
    assert np.array_equal(oracle.rng_draws(0x5EED, 97, 16, "normal"), g["rng_normal_5eed_97"])


# ------------------------------------------------------------------ live (_ref present)
@live
@pytest.mark.parametrize("kind,N,n,K,seed,pieces", [
    ("maxaffine-uniform", 90, 6, None, 31, 8),
    ("sqnorm-uniform", 77, 5, None, 32, 0),
    ("lse-uniform", 45, 12, None, 33, 20),
    ("quadratic", 60, 4, 6, 34, 0),
    ("quadratic", 56, 3, 2, 35, 0),
])
def test_live_operators_and_sigma(oracle, kind, N, n, K, seed, pieces):
    X, _ = oracle.gen_instance(kind, N, n, 0.2, seed, pieces)
    rng = np.random.default_rng(seed)
    yy, xi = rng.standard_normal(N), rng.standard_normal((N, n))
    th = rng.random(N * (N - N // (K or N)) + N)
    if K is None:
        a, b, s = oracle.apply_C(X, yy, xi), oracle.apply_C_T(X, th), oracle.sigma_C(X)
    else:
        a, b, s = oracle.apply_C_k(X, K, yy, xi), oracle.apply_C_T_k(X, K, th), oracle.sigma_C_k(X, K)
    assert np.array_equal(a, R.apply_C(X, yy, xi, K))
    rb = R.apply_C_T(X, th, K)
    assert np.array_equal(b[0], rb[0]) and np.array_equal(b[1], rb[1])
    rs = R.sigma(X, "C", K)
    assert s[1:] == rs[1:] and s[0] == pytest.approx(rs[0], rel=1e-13)


@live
@pytest.mark.parametrize("kind,N,n,seed,pieces,iters,mom,kw", [
    ("maxaffine-uniform", 120, 10, 41, 20, 40, True, {}),
    ("lse-uniform", 70, 20, 42, 50, 30, True, {}),
    ("sqnorm-uniform", 100, 5, 43, 0, 60, False, {}),                      # DGA
    ("sqnorm-uniform", 90, 3, 44, 0, 400, True, dict(gap_norm_tol=1e9, infeas_norm_tol=1e9,
                                                     B_theta=1e-5)),       # restarts
    ("maxaffine-uniform", 200, 10, 45, 20, 5000, True, dict(gap_norm_tol=1e-4)),  # cfg 2 rule
])
def test_live_singleton_papg_matches_reference(oracle, kind, N, n, seed, pieces, iters, mom, kw):
    """The hot path: the reference's papg_solve on Partition{N, 1} against the oracle."""
    X, y = oracle.gen_instance(kind, N, n, 0.1, seed, pieces)
    P = R.prepare(X, y)
    base = dict(gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
    base.update(kw)
    r = R.papg(X, P.ys, feas_y=P.feas_y, feas_xi=P.feas_xi, max_iters=iters, use_momentum=mom,
               **base)
    o = oracle.papg(X, P.ys, max_iters=iters, use_momentum=mom, sigma_C=r.sigma_C, **base)
    assert (o.iters, o.reason, o.restarts, o.saturated) == (r.iters, r.reason, r.restarts,
                                                            r.saturated)
    assert np.linalg.norm(r.theta) > 0
    assert rel(o.theta, r.theta) <= 1e-13 and rel(o.y, r.y) <= 1e-13 and rel(o.xi, r.xi) <= 1e-13
    hist_close(o.history, r.history, 1e-11)
    assert o.g_final == pytest.approx(r.g_final, rel=1e-12, abs=1e-13)
    assert o.delta_estimate == pytest.approx(r.delta_estimate, rel=1e-10, abs=1e-12)
    assert o.B_theta == r.B_theta


@live
def test_live_general_k_and_alcc(oracle):
    X, y = oracle.gen_instance("quadratic", 54, 3, 0.4, 51)
    P = R.prepare(X, y)
    inner = dict(max_outer=6, mapg_cap=1000)
    r = R.papg(X, P.ys, K=3, feas_y=P.feas_y, feas_xi=P.feas_xi, inner=inner, max_iters=8,
               gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
    o = oracle.papg_k(X, P.ys, 3, P.feas_y, P.feas_xi, inner=inner, sigma_C=r.sigma_C, max_iters=8,
                      gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
    assert o.iters == r.iters and rel(o.theta, r.theta) <= 1e-10 and rel(o.y, r.y) <= 1e-10
    s1, s2 = R.sigma(X, "A1"), R.sigma(X, "A2")
    kw = dict(gamma=1e-3, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, warm_y=P.feas_y, warm_xi=P.feas_xi,
              max_outer=5, mapg_cap=1500)
    a = R.alcc(X, P.ys, **kw)
    b = oracle.alcc(X, P.ys, sigma_A1=s1[0], sigma_A2=s2[0], **kw)
    assert (a.outer_iters, a.mapg_iters_total, a.reason) == (b.outer_iters, b.mapg_iters_total,
                                                             b.reason)
    assert rel(b.y, a.y) <= 1e-12 and rel(b.xi, a.xi) <= 1e-12


@live
def test_live_reference_error_conventions():
    """validate_dataset / make_partition errors are std::invalid_argument."""
    X = np.array([[0.0, 1.0], [0.0, 1.0], [2.0, 3.0], [4.0, 5.0]])
    with pytest.raises(ValueError, match="duplicate x rows"):
        R.validate(X, np.zeros(4))
    Xg, yg = R.gen_instance("quadratic", 24, 3, 0.1, 2)
    with pytest.raises(ValueError, match="block size"):
        R.apply_C(Xg, np.zeros(24), np.zeros((24, 3)), K=12)  # nbar = 2 < n + 1


@live
def test_fixtures_are_current():
    """The committed fixtures are what the compiled reference produces now."""
    g = np.load(os.path.join(GOLDEN, "ref_papg_singleton.npz"))
    i = 0
    iters, _, gt, ft, B, mom = g[f"meta{i}"]
    feas = g[f"feas{i}"]
    N = g[f"X{i}"].shape[0]
    r = R.papg(g[f"X{i}"], g[f"ys{i}"], feas_y=feas[:N], feas_xi=feas[N:], max_iters=int(iters),
               gap_norm_tol=float(gt), infeas_norm_tol=float(ft), B_theta=float(B),
               use_momentum=bool(mom))
    assert np.array_equal(r.theta, g[f"theta{i}"]) and np.array_equal(r.y, g[f"y{i}"])


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("CRB_SLOW_TESTS"), reason="1-2 minutes of oracle time; "
                    "set CRB_SLOW_TESTS=1 (the GPU suite checks the same fixture on the device)")
def test_oracle_reproduces_reference_at_baseline_config_1(oracle):
    """BASELINE config 1 (N = 1000, n = 5, 2000 iterations): the oracle against the reference's
    own run (tests/golden/ref_baseline_cfg1.npz, scripts/make_ref_baseline_golden.py)."""
    path = os.path.join(GOLDEN, "ref_baseline_cfg1.npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated")
    g = np.load(path)
    X, _ = oracle.gen_instance("sqnorm-uniform", 1000, 5, 0.1, 1, 0)
    iters, gt, ft = g["meta"]
    r = oracle.papg(X, g["ys"], max_iters=int(iters), gap_norm_tol=float(gt),
                    infeas_norm_tol=float(ft), sigma_C=float(g["scal"][4]),
                    threads=os.cpu_count() or 1)
    assert r.iters == int(g["iters"][0]) == 2000
    N = 1000
    cross = r.theta[: N * (N - 1)].reshape(N, N - 1)
    assert rel(cross[g["rows"]], g["theta_rows"]) <= 1e-12
    assert rel(r.theta, np.zeros(1)) == pytest.approx(float(g["theta_norm"]), rel=1e-12)
    assert rel(r.y, g["y"]) <= 1e-12 and rel(r.xi, g["xi"]) <= 1e-11
    hist_close(r.history, g["hist"], 1e-9)


@live
def test_live_prepare_and_size_edge_cases(oracle):
    """Edge cases of preprocess.cpp / testgen.cpp: rank-deficient design (constant-fit
    fallback, preprocess.cpp:27-31), exactly affine data, the minimal N = n + 1, N < n + 1."""
    rng = np.random.default_rng(0)
    x1 = rng.standard_normal(30)
    X = np.stack([x1, 2 * x1, rng.standard_normal(30)], 1)  # columns 1 and 2 collinear
    y = rng.standard_normal(30)
    po, pr = oracle.prepare(X, y), R.prepare(X, y)
    assert np.array_equal(pr.slope, np.zeros(3)) and np.array_equal(po.slope, pr.slope)
    assert po.intercept == pytest.approx(pr.intercept, rel=1e-14)
    assert np.abs(po.ys - pr.ys).max() <= 1e-13 and po.shift == pytest.approx(pr.shift, rel=1e-14)
    X = rng.standard_normal((20, 2))
    y = 0.5 + X @ np.array([1.0, -2.0])  # affine: the fit is exact
    po, pr = oracle.prepare(X, y), R.prepare(X, y)
    assert po.Bbar_y == pytest.approx(pr.Bbar_y, rel=1e-9)
    assert po.shift == pytest.approx(pr.shift, rel=1e-12)
    X, y = rng.standard_normal((4, 3)), rng.standard_normal(4)  # N = n + 1
    pr = R.prepare(X, y)
    r = R.papg(X, pr.ys, feas_y=pr.feas_y, feas_xi=pr.feas_xi, max_iters=20, gap_norm_tol=-1.0,
               infeas_norm_tol=-1.0)
    o = oracle.papg(X, pr.ys, max_iters=20, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                    sigma_C=r.sigma_C)
    assert np.linalg.norm(r.theta) > 0 and rel(o.theta, r.theta) <= 1e-13 and rel(o.y, r.y) <= 1e-13
    with pytest.raises(ValueError, match="N >= n"):
        R.gen_instance("quadratic", 3, 3, 0.1, 1)
    with pytest.raises(ValueError):
        oracle.gen_instance("quadratic", 3, 3, 0.1, 1)


@pytest.mark.skipif(not (R.available() and R.available_sequential()),
                    reason="oracle/_ref builds absent")
def test_reference_results_do_not_depend_on_the_stand_ins_summation_order(oracle):
    """Eigen is replaced by oracle/eigen_shim in the compiled reference. Its reductions
    (norm, dot: 8 partial sums) are the one place where a real Eigen build could differ in
    the last bits; the second build sums left to right instead. The reference's trajectory
    moves by rounding only between the two (and the oracle agrees with both), so the choice
    of summation order in the stand-in does not affect what is pinned."""
    X, y = oracle.gen_instance("maxaffine-uniform", 160, 10, 0.1, 77, 20)
    P = R.prepare(X, y)
    kw = dict(feas_y=P.feas_y, feas_xi=P.feas_xi, max_iters=5000, gap_norm_tol=1e-4,
              infeas_norm_tol=1e-1)
    a = R.papg(X, P.ys, **kw)
    b = R.papg(X, P.ys, sequential=True, **kw)
    assert (a.iters, a.reason, a.restarts) == (b.iters, b.reason, b.restarts)
    assert a.reason == "thresholds" and np.linalg.norm(a.theta) > 0
    assert rel(b.theta, a.theta) <= 1e-13 and rel(b.y, a.y) <= 1e-13
    assert b.sigma_C == pytest.approx(a.sigma_C, rel=1e-13)
    hist_close(b.history, a.history, 1e-11)
    o = oracle.papg(X, P.ys, max_iters=5000, gap_norm_tol=1e-4, infeas_norm_tol=1e-1,
                    sigma_C=b.sigma_C)
    assert o.iters == b.iters and rel(o.theta, b.theta) <= 1e-13

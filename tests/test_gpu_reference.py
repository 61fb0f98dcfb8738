"""GPU parity against the REFERENCE's own code (not the oracle restatement).

  * tests/golden/ref_*.npz: outputs of the reference's proj/core sources compiled
    unmodified in the build container (oracle/Makefile target `ref`,
    scripts/make_ref_golden.py); the CUDA path is compared with them directly.
  * when the prebuilt oracle/_ref/libcvxreg_ref.so travelled to this box, the
    reference itself is run here on mid-size seeded instances and compared live.

Tolerances are BASELINE.json north_star's: per-pair residuals and theta after k
iterations within 1e-12 relative, fitted y within 1e-8, identical iteration
counts (and termination reasons, restart counts). sigma_max(C) is the
reference's own estimate, injected into the GPU solve; the device power loop
is compared with it separately (same step count, 1e-10).
"""
import os

import numpy as np
import pytest

import paper_1407_7220_b200 as crb
from oracle import ref as R

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
live = pytest.mark.skipif(not R.available(), reason="oracle/_ref not shipped to this box")
REASON = {"thresholds": 0, "iter_budget": 1, "time_budget": 2, "error": 3}


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def gpu_papg(X, ys, *, momentum=True, theta0=None, partition=None, **kw):
    cfg = crb.PapgConfig(**kw)
    with crb.DualSolver(X, ys, cfg.gamma) as s:
        if partition is not None:
            K, feas_y, feas_xi = partition
            s.set_partition(K, crb.PrimalPoint(feas_y, feas_xi), cfg.inner)
        s.begin(cfg, momentum, theta0)
        stopped = False
        while not stopped:
            _, stopped = s.iterate(1 << 40)
        res, y, xi, hist = s.finish()
        return dict(res=res, y=y, xi=xi, hist=hist, theta=s.theta(), rows=s.rows())


def hist_close(h, g, rtol):
    h, g = np.asarray(h)[:, :7], np.asarray(g)[:, :7]
    assert h.shape[0] == g.shape[0]
    for col in range(1, 7):
        scale = max(np.abs(g[:, col]).max(), 1e-300)
        assert np.abs(h[:, col] - g[:, col]).max() <= rtol * scale, col


@pytest.mark.parametrize("small", ["1", "0"])
def test_singleton_papg_matches_reference_fixtures(monkeypatch, small):
    """Every reference fixture on the persistent small-N loop and on the TMA/DMMA sweep."""
    monkeypatch.setenv("CRB_SMALL", small)
    g = np.load(os.path.join(GOLDEN, "ref_papg_singleton.npz"))
    worst = dict(theta=0.0, rows=0.0, y=0.0)
    for i in range(int(g["count"])):
        X, ys = g[f"X{i}"], g[f"ys{i}"]
        iters, sigma, gt, ft, B, mom = g[f"meta{i}"]
        r = gpu_papg(X, ys, momentum=bool(mom), max_iters=int(iters), sigma_C=float(sigma),
                     gap_norm_tol=float(gt), infeas_norm_tol=float(ft), B_theta=float(B))
        k, restarts, reason, saturated = (int(v) for v in g[f"iters{i}"])
        assert (r["res"].iters, r["res"].restarts, r["res"].reason) == (k, restarts, reason), i
        assert bool(r["res"].saturated) == bool(saturated)
        e_theta, e_y = rel(r["theta"], g[f"theta{i}"]), rel(r["y"], g[f"y{i}"])
        assert e_theta <= 1e-12, (i, e_theta)
        assert e_y <= 1e-8 and rel(r["xi"], g[f"xi{i}"]) <= 1e-8, (i, e_y)
        worst["theta"], worst["y"] = max(worst["theta"], e_theta), max(worst["y"], e_y)
        if g[f"c_eta{i}"].size:  # per-pair residuals of the k-th iteration
            e_rows = rel(r["rows"], g[f"c_eta{i}"])
            assert e_rows <= 1e-12, (i, e_rows)
            worst["rows"] = max(worst["rows"], e_rows)
        hist_close(r["hist"], g[f"hist{i}"], 1e-9)
        gf, de, Bt, Lg = g[f"scal{i}"]
        assert r["res"].g_final == pytest.approx(gf, rel=1e-9, abs=1e-12)
        assert r["res"].delta_estimate == pytest.approx(de, rel=1e-8, abs=1e-10)
        assert r["res"].B_theta == Bt
    print(f"GPU vs reference fixtures (CRB_SMALL={small}): worst {worst}")


def test_warm_start_matches_reference_fixture():
    g = np.load(os.path.join(GOLDEN, "ref_papg_singleton.npz"))
    i = 1
    r = gpu_papg(g[f"X{i}"], g[f"ys{i}"], max_iters=20, sigma_C=float(g[f"meta{i}"][1]),
                 gap_norm_tol=-1.0, infeas_norm_tol=-1.0, B_theta=20.0, theta0=g["warm_theta0"])
    assert rel(r["theta"], g["warm_theta"]) <= 1e-12 and rel(r["y"], g["warm_y"]) <= 1e-8
    hist_close(r["hist"], g["warm_hist"], 1e-9)


def test_sigma_power_loop_matches_reference_fixtures():
    g = np.load(os.path.join(GOLDEN, "ref_papg_singleton.npz"))
    for i in range(int(g["count"])):
        with crb.DualSolver(g[f"X{i}"], g[f"ys{i}"]) as s:
            sg, it, cv = s.sigma_C()
        assert (it, int(cv)) == (int(g[f"sigma{i}"][1]), int(g[f"sigma{i}"][2])), i
        assert sg == pytest.approx(g[f"sigma{i}"][0], rel=1e-10)


def test_general_k_matches_reference_fixtures():
    """f2: the reference's default solver (K < N blocks, ALCC block solves)."""
    g = np.load(os.path.join(GOLDEN, "ref_papg_general.npz"))
    for i in range(int(g["count"])):
        X, ys, feas = g[f"X{i}"], g[f"ys{i}"], g[f"feas{i}"]
        N = X.shape[0]
        iters, sigma, K, mo, cap = g[f"meta{i}"]
        r = gpu_papg(X, ys, partition=(int(K), feas[:N], feas[N:]), max_iters=int(iters),
                     sigma_C=float(sigma), K=int(K), gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                     inner=crb.AlccConfig(max_outer=int(mo), mapg_cap=int(cap)))
        assert r["res"].iters == int(iters)
        assert rel(r["theta"], g[f"theta{i}"]) <= 1e-9, rel(r["theta"], g[f"theta{i}"])
        assert rel(r["y"], g[f"y{i}"]) <= 1e-8
        hist_close(r["hist"], g[f"hist{i}"], 1e-7)
        with crb.DualSolver(X, ys) as s:
            s.set_partition(int(K), crb.PrimalPoint(feas[:N], feas[N:]))
            sg, it, cv = s.sigma_C()
        assert (it, int(cv)) == (int(g[f"sigma{i}"][1]), int(g[f"sigma{i}"][2]))
        assert sg == pytest.approx(g[f"sigma{i}"][0], rel=1e-10)


def test_alcc_matches_reference_fixtures():
    """f1: the reference's alcc_solve."""
    g = np.load(os.path.join(GOLDEN, "ref_alcc.npz"))
    for i in range(int(g["count"])):
        X, ys, feas = g[f"X{i}"], g[f"ys{i}"], g[f"feas{i}"]
        N = X.shape[0]
        mo, cap, By, Bxi, s1, s2, it1, it2 = g[f"meta{i}"]
        cfg = crb.AlccConfig(sigma_A1=s1, sigma_A2=s2, max_outer=int(mo), mapg_cap=int(cap))
        bounds = crb.ProblemBounds(10.0 * np.sqrt(N), By, Bxi, 1e-3)
        with crb.DualSolver(X, ys, 1e-3) as s:
            res, y, xi, hist, mi = s.alcc(cfg, bounds, crb.PrimalPoint(feas[:N], feas[N:]))
            mult = s.alcc_multiplier()
            sa1, sa2 = s.sigma_A(1), s.sigma_A(2)
        outer, mapg, reason, cert, infeas, gap, obj = g[f"scal{i}"]
        assert (res.outer_iters, res.mapg_iters_total, res.reason) == (int(outer), int(mapg),
                                                                       int(reason))
        assert rel(y, g[f"y{i}"]) <= 1e-10 and rel(xi, g[f"xi{i}"]) <= 1e-10
        assert rel(mult, g[f"mult{i}"]) <= 1e-7
        assert res.certified_gap == pytest.approx(cert, rel=1e-8)
        assert res.objective == pytest.approx(obj, rel=1e-8)
        assert (sa1[1], sa2[1]) == (int(it1), int(it2))
        assert sa1[0] == pytest.approx(s1, rel=1e-10) and sa2[0] == pytest.approx(s2, rel=1e-10)


def test_metric_sweeps_match_reference_fixtures():
    """f3: metrics.cpp on the device against the reference's values."""
    g = np.load(os.path.join(GOLDEN, "ref_operators.npz"))
    X, yy, xi = g["X"], g["yy"], g["xi"]
    N = X.shape[0]
    th = g[f"theta_K{N}"]
    with crb.DualSolver(X, np.zeros(N)) as s:
        # theta1 of the handle := th (inside Q2: nonnegative, |th| < 10 sqrt(N))
        s.begin(crb.PapgConfig(max_iters=1, sigma_C=10.0), True, th)
        inf = s.infeasibility(yy, xi)
        gap = s.duality_gap(yy, xi)
        ev = s.evaluate_estimator(yy, xi, X[3] + 0.1)[0]
        rep = s.repair_feasibility(yy, xi)
    got = np.array([inf[0], inf[1], gap[0], gap[1], ev])
    assert np.allclose(got, g["metrics"], rtol=1e-12)
    assert np.allclose(rep, g["repair"], rtol=1e-13, atol=1e-14)


# ------------------------------------------------------------------ live reference runs
@live
@pytest.mark.parametrize("kind,N,n,pieces,noise,iters,small", [
    ("maxaffine-uniform", 700, 10, 20, 0.1, 30, "0"),   # cfg 2's kind on the DMMA sweep
    ("lse-uniform", 500, 20, 50, 0.05, 20, "0"),        # cfg 3's kind
    ("sqnorm-uniform", 600, 5, 0, 0.1, 40, "1"),        # cfg 1's kind, persistent loop
])
def test_live_reference_singleton_parity(monkeypatch, kind, N, n, pieces, noise, iters, small):
    """The reference's papg_solve (Partition{N, 1}) run on this box against the CUDA path."""
    from oracle import oracle as O

    monkeypatch.setenv("CRB_SMALL", small)
    X, y = O.gen_instance(kind, N, n, noise, 70 + n, pieces)
    P = R.prepare(X, y)
    r = R.papg(X, P.ys, feas_y=P.feas_y, feas_xi=P.feas_xi, max_iters=iters, gap_norm_tol=-1.0,
               infeas_norm_tol=-1.0, threads=os.cpu_count() or 1)
    g = gpu_papg(X, P.ys, max_iters=iters, sigma_C=r.sigma_C, gap_norm_tol=-1.0,
                 infeas_norm_tol=-1.0)
    assert g["res"].iters == r.iters == iters
    e = rel(g["theta"], r.theta), rel(g["y"], r.y)
    print(f"live reference {kind} N={N} n={n}: |dtheta|/|theta|={e[0]:.2e} |dy|/|y|={e[1]:.2e}")
    assert e[0] <= 1e-12 and e[1] <= 1e-8
    hist_close(g["hist"], r.history, 1e-9)
    with crb.DualSolver(X, P.ys) as s:
        sg, it, _ = s.sigma_C()
    assert sg == pytest.approx(r.sigma_C, rel=1e-10)


@live
def test_live_reference_to_tolerance(monkeypatch):
    """cfg 2's stopping rule on a mid-size instance: same iteration count and reason."""
    from oracle import oracle as O

    monkeypatch.setenv("CRB_SMALL", "0")
    X, y = O.gen_instance("maxaffine-uniform", 1200, 10, 0.1, 1, 20)
    P = R.prepare(X, y)
    kw = dict(gap_norm_tol=1e-4, infeas_norm_tol=1e-1, max_iters=5000)
    r = R.papg(X, P.ys, feas_y=P.feas_y, feas_xi=P.feas_xi, threads=os.cpu_count() or 1, **kw)
    g = gpu_papg(X, P.ys, sigma_C=r.sigma_C, **kw)
    assert r.reason == "thresholds"
    assert (g["res"].iters, g["res"].reason, g["res"].restarts) == (r.iters, 0, r.restarts)
    assert rel(g["theta"], r.theta) <= 1e-12 and rel(g["y"], r.y) <= 1e-8


# ------------------------------------------- BASELINE configurations, reference fixtures
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_baseline_config_matches_the_compiled_reference(monkeypatch, name):
    """BASELINE configs 1-3 against tests/golden/ref_baseline_<cfg>.npz: the reference's own
    papg_solve run in the build container (scripts/make_ref_baseline_golden.py; config 1 for
    its 2000 iterations, config 2 to its tolerance, config 3 for 10 iterations). The fixture
    keeps y, xi, the history, the decisions, sigma_C and 12 sampled rows of theta."""
    import bench
    from oracle import oracle as O

    path = os.path.join(GOLDEN, f"ref_baseline_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = np.load(path)
    cfg = bench.CONFIGS[name]
    N, n = cfg["N"], cfg["n"]
    X, _ = O.gen_instance(cfg["kind"], N, n, cfg["noise"], 1, cfg["pieces"])
    iters, gt, ft = g["meta"]
    g_final, delta, B_theta, L_g, sigma = g["scal"]
    with crb.DualSolver(X, g["ys"]) as s:
        sg, _, _ = s.sigma_C()
        assert sg == pytest.approx(sigma, rel=1e-10)  # device power loop vs the reference's
        pc = crb.PapgConfig(max_iters=int(iters), gap_norm_tol=float(gt),
                            infeas_norm_tol=float(ft), sigma_C=float(sigma))
        s.begin(pc)
        stopped = False
        while not stopped:
            _, stopped = s.iterate(1 << 40)
        res, y, xi, hist = s.finish()
        k, restarts, reason, saturated = (int(v) for v in g["iters"])
        assert (res.iters, res.restarts, res.reason, int(bool(res.saturated))) == \
            (k, restarts, reason, saturated)
        e_y, e_xi = rel(y, g["y"]), rel(xi, g["xi"])
        num = den = 0.0
        for r, want in zip(g["rows"], g["theta_rows"]):
            got = s.theta_rows(int(r), int(r) + 1)
            num += np.sum((got[: N - 1] - want) ** 2)
            den += np.sum(want ** 2)
            pos = got[N - 1:]
        e_theta = np.sqrt(num / max(den, 1e-300))
        e_pos = rel(pos, g["theta_pos"]) if np.linalg.norm(g["theta_pos"]) > 0 else \
            np.linalg.norm(pos)
    print(f"{name} vs compiled reference: iterations {res.iters}, |dtheta|/|theta| (sampled rows) "
          f"{e_theta:.2e}, pos rows {e_pos:.2e}, |dy|/|y| {e_y:.2e}, |dxi|/|xi| {e_xi:.2e}")
    assert den > 0 and e_theta <= 1e-12 and e_pos <= 1e-12
    assert e_y <= 1e-8 and e_xi <= 1e-8
    hist_close(hist, g["hist"], 1e-9)
    assert res.g_final == pytest.approx(g_final, rel=1e-9)
    assert res.delta_estimate == pytest.approx(delta, rel=1e-7, abs=1e-9)
    assert res.B_theta == B_theta


@live
def test_live_reference_general_k_and_alcc():
    """f2 / f1 against the reference run on this box: papg_solve with K = 4 blocks of 60
    points (block QPs by the reference's ALCC) and the standalone alcc_solve at N = 150."""
    from oracle import oracle as O

    X, y = O.gen_instance("maxaffine-uniform", 240, 4, 0.2, 61, 8)
    P = R.prepare(X, y)
    inner = dict(max_outer=8, mapg_cap=1500)
    r = R.papg(X, P.ys, K=4, feas_y=P.feas_y, feas_xi=P.feas_xi, inner=inner, max_iters=10,
               gap_norm_tol=-1.0, infeas_norm_tol=-1.0, threads=os.cpu_count() or 1)
    g = gpu_papg(X, P.ys, partition=(4, P.feas_y, P.feas_xi), max_iters=10, sigma_C=r.sigma_C,
                 K=4, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, inner=crb.AlccConfig(**inner))
    assert g["res"].iters == r.iters == 10
    e = rel(g["theta"], r.theta), rel(g["y"], r.y)
    print(f"live reference general K=4 N=240: |dtheta|/|theta|={e[0]:.2e} |dy|/|y|={e[1]:.2e}")
    assert e[0] <= 1e-9 and e[1] <= 1e-8
    hist_close(g["hist"], r.history, 1e-7)

    X, y = O.gen_instance("sqnorm-uniform", 150, 3, 0.2, 62, 0)
    P = R.prepare(X, y)
    s1, s2 = R.sigma(X, "A1"), R.sigma(X, "A2")
    a = R.alcc(X, P.ys, gamma=1e-3, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, warm_y=P.feas_y,
               warm_xi=P.feas_xi, max_outer=5, mapg_cap=1500, want_multiplier=True)
    cfg = crb.AlccConfig(sigma_A1=s1[0], sigma_A2=s2[0], max_outer=5, mapg_cap=1500)
    bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, 1e-3)
    with crb.DualSolver(X, P.ys, 1e-3) as s:
        res, yg, xig, hist, mi = s.alcc(cfg, bounds, crb.PrimalPoint(P.feas_y, P.feas_xi))
        mult = s.alcc_multiplier()
    assert (res.outer_iters, res.mapg_iters_total, res.reason) == \
        (a.outer_iters, a.mapg_iters_total, REASON[a.reason])
    e = rel(yg, a.y), rel(mult, a.multiplier)
    print(f"live reference ALCC N=150: outer {a.outer_iters}, MAPG {a.mapg_iters_total}, "
          f"|dy|/|y|={e[0]:.2e} |dlambda|/|lambda|={e[1]:.2e}")
    assert e[0] <= 1e-10 and rel(xig, a.xi) <= 1e-10 and e[1] <= 1e-7

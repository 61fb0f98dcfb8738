"""GPU parity of the standalone ALCC (cr_alcc_solve)
against the oracle restatement of alcc_solve (alcc.cpp:54-208, engines.cpp:57-106).

Tolerances: same outer-step count, termination reason and MAPG iteration
count per outer step; the primal point within 1e-10 relative (normwise), the
multiplier lambda = mu (theta - row)_+ within 1e-7 relative (its active entries
are differences of nearly equal O(1) numbers, so last-bit differences of the
residual rows are amplified), history scalars within 1e-8. The spectral
norms sigma(A1), sigma(A2) are injected identically into both paths except in
the sigma tests themselves.
"""
import numpy as np
import pytest

import paper_1407_7220_b200 as crb

pytestmark = pytest.mark.gpu

REASON = {"thresholds": 0, "iter_budget": 1, "time_budget": 2, "error": 3}


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def problem(O, kind, N, n, noise, seed, pieces=0):
    X, y = O.gen_instance(kind, N, n, noise, seed, pieces)
    return X, O.prepare(X, y, 1e-3)


def run_both(O, X, P, warm_y=None, warm_xi=None, **kw):
    s1 = O.sigma_A(X, 1)[0]
    s2 = O.sigma_A(X, 2)[0]
    wy = P.feas_y if warm_y is None else warm_y
    wx = P.feas_xi if warm_xi is None else warm_xi
    o = O.alcc(X, P.ys, gamma=P.gamma, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, warm_y=wy,
               warm_xi=wx, sigma_A1=s1, sigma_A2=s2, want_multiplier=True, **kw)
    cfg = crb.AlccConfig(sigma_A1=s1, sigma_A2=s2, **kw)
    bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma)
    with crb.DualSolver(X, P.ys, P.gamma) as s:
        res, y, xi, hist, mi = s.alcc(cfg, bounds, crb.PrimalPoint(wy, wx))
        mult = s.alcc_multiplier() if res.outer_iters > 0 else None
    return o, dict(res=res, y=y, xi=xi, hist=hist, mapg=mi, mult=mult)


def assert_alcc_parity(o, g, tol_y=1e-10, tol_mult=1e-7, hist_rtol=1e-8):
    r = g["res"]
    assert r.outer_iters == o.outer_iters
    assert r.reason == REASON[o.reason]
    assert list(g["mapg"]) == list(o.mapg_iters)
    assert r.mapg_iters_total == o.mapg_iters_total
    assert rel(g["y"], o.y) <= tol_y, rel(g["y"], o.y)
    assert rel(g["xi"], o.xi.reshape(-1)) <= tol_y, rel(g["xi"], o.xi.reshape(-1))
    if o.outer_iters > 0:
        if tol_mult is not None:
            assert rel(g["mult"], o.multiplier) <= tol_mult, rel(g["mult"], o.multiplier)
        np.testing.assert_allclose(g["hist"][:, [0, 1, 2, 3, 4]], o.history[:, [0, 1, 2, 3, 4]],
                                   rtol=hist_rtol, atol=1e-13)
        np.testing.assert_allclose(g["hist"][:, 5], o.history[:, 5], rtol=10 * hist_rtol,
                                   atol=hist_rtol / 100 * max(1.0, np.abs(o.history[:, 5]).max()))
        scale = max(1.0, abs(o.objective))
        assert abs(r.certified_gap - o.certified_gap) <= hist_rtol * scale
        assert r.infeas_raw == pytest.approx(o.infeas_raw, rel=hist_rtol, abs=1e-13)
    assert r.objective == pytest.approx(o.objective, rel=100 * tol_y, abs=1e-14)


@pytest.mark.parametrize("N,n,seed,kind,max_outer", [
    (40, 1, 1, "sqnorm-uniform", 6),
    (64, 2, 3, "sqnorm-uniform", 6),
    (50, 3, 5, "maxaffine-uniform", 5),
    (70, 5, 7, "lse-uniform", 5),
    (45, 7, 9, "sqnorm-uniform", 4),
    (33, 12, 2, "maxaffine-uniform", 4),
    (37, 20, 4, "sqnorm-uniform", 3),
])
def test_alcc_parity(oracle, N, n, seed, kind, max_outer):
    X, P = problem(oracle, kind, N, n, 0.2, seed, 0 if kind == "sqnorm-uniform" else 3)
    o, g = run_both(oracle, X, P, max_outer=max_outer, mapg_cap=1000)
    assert_alcc_parity(o, g)


def test_alcc_parity_long_inner_runs(oracle):
    """thousands of accelerated inner steps at mu = c^3: last-bit differences of
    the two summation orders grow with the inner condition number (sigma^2 mu),
    measured 1e-16 -> 1e-13 -> 6e-8 over 1 -> 1478 -> 4000 MAPG steps (the
    history's small late entries up to 1.5e-4 relative). The
    iteration counts and the stop decisions still agree exactly."""
    X, P = problem(oracle, "maxaffine-uniform", 50, 3, 0.2, 5, 3)
    o, g = run_both(oracle, X, P, max_outer=5, mapg_cap=4000)
    # lambda = mu (theta - row)_+ at mu = 125 turns the 6e-8 point difference
    # into ~1e-3 relative on its small active entries: compared through the
    # history (gap = lambda . row) instead
    assert_alcc_parity(o, g, tol_y=1e-6, tol_mult=None, hist_rtol=1e-3)


def test_alcc_parity_dmma_sweep(oracle):
    X, P = problem(oracle, "sqnorm-uniform", 90, 4, 0.2, 13)
    o, g = run_both(oracle, X, P, max_outer=5, mapg_cap=1000)
    assert_alcc_parity(o, g)


def test_alcc_thresholds_stop(oracle):
    """default tolerances: the standalone stop (alcc.cpp:160-165) fires"""
    X, P = problem(oracle, "sqnorm-uniform", 60, 2, 0.1, 3)
    o, g = run_both(oracle, X, P, max_outer=30)
    assert o.reason == "thresholds"
    assert_alcc_parity(o, g)


def test_alcc_projected_warm_start(oracle):
    """a warm point outside both balls is projected first (alcc.cpp:68-69)"""
    X, P = problem(oracle, "sqnorm-uniform", 48, 2, 0.2, 21)
    wy = P.ys + 10.0 * P.Bbar_y
    wx = np.full(X.size, 5.0 * P.Bbar_xi)
    o, g = run_both(oracle, X, P, warm_y=wy, warm_xi=wx, max_outer=4, mapg_cap=1000)
    assert_alcc_parity(o, g)


def test_alcc_zero_outer(oracle):
    X, P = problem(oracle, "sqnorm-uniform", 30, 2, 0.2, 2)
    wy = P.ys + 10.0 * P.Bbar_y
    o, g = run_both(oracle, X, P, warm_y=wy, max_outer=0)
    assert g["res"].outer_iters == 0
    assert rel(g["y"], o.y) <= 1e-14


def test_alcc_mapg_cap(oracle):
    """tiny cap: every MAPG call runs to l_max (engines.cpp:105)"""
    X, P = problem(oracle, "sqnorm-uniform", 40, 2, 0.3, 8)
    o, g = run_both(oracle, X, P, max_outer=4, mapg_cap=12, infeas_norm_tol=0.0)
    assert g["res"].hit_cap_any
    assert_alcc_parity(o, g)


def test_sigma_A_matches_oracle(oracle):
    for N, n, seed in ((40, 2, 1), (77, 5, 2), (50, 13, 3)):
        X, _ = oracle.gen_instance("sqnorm-uniform", N, n, 0.1, seed)
        with crb.DualSolver(X, np.zeros(N)) as s:
            for which in (1, 2):
                sg, it, cv = s.sigma_A(which)
                so, ito, cvo = oracle.sigma_A(X, which)
                assert it == ito and cv == cvo
                assert sg == pytest.approx(so, rel=1e-10)


def test_alcc_estimated_sigmas(oracle):
    """no injection: both paths estimate sigma(A1), sigma(A2) themselves"""
    X, P = problem(oracle, "sqnorm-uniform", 52, 3, 0.2, 4)
    o = oracle.alcc(X, P.ys, gamma=P.gamma, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi,
                    warm_y=P.feas_y, warm_xi=P.feas_xi, max_outer=4, mapg_cap=3000)
    r = crb.alcc_solve(crb.PreparedProblem(crb.Dataset(X, P.ys), P.shift,
                                           crb.PrimalPoint(P.feas_y, P.feas_xi),
                                           crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi,
                                                             P.gamma)),
                       crb.AlccConfig(max_outer=4, mapg_cap=3000))
    assert r.sigma_A1 == pytest.approx(o.sigma_A1, rel=1e-10)
    assert r.sigma_A2 == pytest.approx(o.sigma_A2, rel=1e-10)
    assert r.report.iters == o.outer_iters
    assert list(r.mapg_iters) == list(o.mapg_iters)
    assert rel(r.point.y, o.y) <= 1e-9


def test_alcc_errors(oracle):
    X, P = problem(oracle, "sqnorm-uniform", 20, 2, 0.2, 1)
    bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma)
    warm = crb.PrimalPoint(P.feas_y, P.feas_xi)
    with crb.DualSolver(X, P.ys) as s:
        for bad in (dict(c=1.0), dict(kappa=0.0), dict(mu1=-1.0)):
            with pytest.raises(ValueError):
                s.alcc(crb.AlccConfig(**bad), bounds, warm)
        with pytest.raises(RuntimeError):  # no finished solve yet
            s.alcc_multiplier()
    with crb.DualSolver(X, P.ys, row_begin=0, row_end=10) as s:  # a shard
        with pytest.raises(ValueError):
            s.alcc(crb.AlccConfig(), bounds, warm)


def test_alcc_then_papg_on_one_handle(oracle):
    """an ALCC solve leaves the handle usable for a fresh P-APG solve"""
    X, P = problem(oracle, "sqnorm-uniform", 40, 2, 0.2, 6)
    bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma)
    sig = oracle.sigma_C(X)[0]
    with crb.DualSolver(X, P.ys) as s:
        s.alcc(crb.AlccConfig(max_outer=2), bounds, crb.PrimalPoint(P.feas_y, P.feas_xi))
        cfg = crb.PapgConfig(max_iters=50, sigma_C=sig)
        s.begin(cfg)
        s.iterate(1 << 40)
        res, y, xi, _ = s.finish()
        th = s.theta()
    o = oracle.papg(X, P.ys, max_iters=50, sigma_C=sig)
    assert res.iters == o.iters
    assert rel(th, o.theta) <= 1e-12


def test_alcc_full_size_consistency(oracle):
    """N = 3000: the reported infeasibility equals the metric sweep at the
    returned point, multipliers are >= 0 and vanish where rows are slack."""
    X, P = problem(oracle, "sqnorm-uniform", 3000, 4, 0.2, 31)
    bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma)
    with crb.DualSolver(X, P.ys) as s:
        res, y, xi, hist, mi = s.alcc(crb.AlccConfig(max_outer=3, mapg_cap=400), bounds,
                                      crb.PrimalPoint(P.feas_y, P.feas_xi))
        lam = s.alcc_multiplier(0, 200)
        raw, _ = s.infeasibility(y, xi)
    assert res.outer_iters >= 1
    assert raw == pytest.approx(res.infeas_raw, rel=1e-9)
    assert (lam >= 0).all()
    o_inf = oracle.infeasibility(X, y, xi)[0]
    assert raw == pytest.approx(o_inf, rel=1e-9)


def test_alcc_time_budget(oracle):
    """max_seconds below one outer step: stops after the first outer step with
    reason time_budget (alcc.cpp:167-170)"""
    X, P = problem(oracle, "sqnorm-uniform", 40, 2, 0.2, 17)
    bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma)
    with crb.DualSolver(X, P.ys) as s:
        res, y, xi, hist, mi = s.alcc(crb.AlccConfig(max_seconds=1e-9, infeas_norm_tol=0.0),
                                      bounds, crb.PrimalPoint(P.feas_y, P.feas_xi))
    assert res.outer_iters == 1
    assert res.reason == 2

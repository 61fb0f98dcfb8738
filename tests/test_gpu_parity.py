"""GPU parity of the B200 pair-sweep solver against the CPU oracle.

Tolerances (BASELINE.json north_star): after k iterations the dual iterate
theta and the per-pair residuals C eta agree within 1e-12 relative (normwise),
the fitted y within 1e-8 relative, with identical iteration counts and
termination reasons. sigma_max(C) is injected identically into both paths
except in the sigma tests themselves.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_1407_7220_b200 as crb

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
TOL_THETA = 1e-12
TOL_ROWS = 1e-12
TOL_Y = 1e-8


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def gpu_run(X, ys, *, momentum=True, theta0=None, device_rows=None, **kw):
    cfg = crb.PapgConfig(**kw)
    with crb.DualSolver(X, ys, cfg.gamma) as s:
        s.begin(cfg, momentum, theta0)
        stopped = False
        while not stopped:
            _, stopped = s.iterate(1 << 40)
        res, y, xi, hist = s.finish()
        return dict(res=res, y=y, xi=xi, hist=hist, theta=s.theta(), rows=s.rows())


def oracle_run(O, X, ys, *, momentum=True, theta0=None, **kw):
    kw = dict(kw)
    kw.pop("graph_iters", None)
    return O.papg(X, ys, use_momentum=momentum, theta0=theta0, want_c_eta=True, **kw)


def instance(O, kind, N, n, noise, seed, pieces=0):
    X, y = O.gen_instance(kind, N, n, noise, seed, pieces)
    p = O.prepare(X, y)
    return X, p.ys


def assert_parity(g, o, hist_rtol=1e-9):
    assert g["res"].iters == o.iters
    assert g["res"].reason == {"thresholds": 0, "iter_budget": 1, "time_budget": 2,
                               "error": 3}[o.reason]
    assert g["res"].restarts == o.restarts
    assert rel(g["theta"], o.theta) <= TOL_THETA, rel(g["theta"], o.theta)
    assert rel(g["rows"], o.c_eta) <= TOL_ROWS, rel(g["rows"], o.c_eta)
    assert rel(g["y"], o.y) <= TOL_Y, rel(g["y"], o.y)
    assert rel(g["xi"], o.xi.reshape(-1)) <= 1e-8
    h, ho = g["hist"], o.history
    for col in (1, 2, 3, 4):  # objective, reg_objective, infeas_raw, infeas_norm
        assert np.allclose(h[:, col], ho[:, col], rtol=hist_rtol, atol=1e-300)
    for col in (5, 6):  # gap may cross zero: compare against its scale
        scale = np.abs(ho[:, col]).max()
        assert np.abs(h[:, col] - ho[:, col]).max() <= hist_rtol * max(scale, 1e-300)
    assert g["res"].g_final == pytest.approx(o.g_final, rel=1e-9, abs=1e-12)


def test_smoke_parity(oracle):
    X, ys = instance(oracle, "sqnorm-uniform", 300, 5, 0.1, 7)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=60, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    assert_parity(gpu_run(X, ys, **kw), oracle_run(oracle, X, ys, **kw))


def test_golden_fixtures():
    g = np.load(os.path.join(GOLDEN, "papg_small.npz"))
    for i in range(int(g["count"])):
        X, ys = g[f"X{i}"], g[f"ys{i}"]
        it, s, gt, ft, B, mom = g[f"meta{i}"]
        r = gpu_run(X, ys, momentum=bool(mom), max_iters=int(it), sigma_C=float(s),
                    gap_norm_tol=float(gt), infeas_norm_tol=float(ft), B_theta=float(B))
        assert r["res"].iters == int(g[f"iters{i}"][0])
        assert rel(r["theta"], g[f"theta{i}"]) <= TOL_THETA
        assert rel(r["rows"], g[f"c_eta{i}"]) <= TOL_ROWS
        assert rel(r["y"], g[f"y{i}"]) <= TOL_Y
        assert rel(r["xi"], g[f"xi{i}"].reshape(-1)) <= 1e-8


@pytest.mark.parametrize("variant", ["mma", "small"])
@pytest.mark.parametrize("n", list(range(1, 33)))
def test_every_n_every_sweep_path(oracle, monkeypatch, variant, n):
    """Every n on each sweep implementation: the TMA-pipelined DMMA kernel
    (per-kernel iteration) and the persistent small-N loop."""
    monkeypatch.setenv("CRB_SMALL", "1" if variant == "small" else "0")
    N = 67 + 3 * n  # ragged: not a multiple of any strip or tile width
    X, ys = instance(oracle, "maxaffine-uniform", N, n, 0.1, 100 + n, 6)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=15, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    assert_parity(gpu_run(X, ys, **kw), oracle_run(oracle, X, ys, **kw))


@pytest.mark.parametrize("small", ["1", "0"])
def test_config1_full_2000_iterations(oracle, monkeypatch, small):
    """BASELINE config 1: N=1000, n=5, |x|^2 + U[-0.1, 0.1] noise, 2000 iterations
    (persistent small-N loop and per-kernel path)."""
    monkeypatch.setenv("CRB_SMALL", small)
    X, ys = instance(oracle, "sqnorm-uniform", 1000, 5, 0.1, 1)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=2000, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    o = oracle_run(oracle, X, ys, threads=8, **kw)
    g = gpu_run(X, ys, **kw)
    assert_parity(g, o, hist_rtol=1e-8)
    print(f"config1 small={small}: iters={o.iters} theta {rel(g['theta'], o.theta):.2e} "
          f"rows {rel(g['rows'], o.c_eta):.2e} y {rel(g['y'], o.y):.2e}")


@pytest.mark.parametrize("method", ["closed-form", "sweep"])
def test_sigma_C_parity(oracle, monkeypatch, method):
    """Power iteration on C^T C (operators.cpp:302-339): the default O(N n^2)
    closed-form step and the O(N^2 n) pair-sweep step both reproduce the
    oracle's sigma and iteration count."""
    if method == "sweep":
        monkeypatch.setenv("CRB_SIGMA", "sweep")
    for kind, N, n, pieces in [("sqnorm-uniform", 400, 5, 0), ("maxaffine-uniform", 300, 10, 20),
                               ("lse-uniform", 250, 20, 50), ("quadratic", 333, 1, 0),
                               ("exponential", 150, 24, 0)]:
        X, ys = instance(oracle, kind, N, n, 0.1, 3, pieces)
        so, ito, co = oracle.sigma_C(X)
        with crb.DualSolver(X, ys) as d:
            sg, itg, cg = d.sigma_C()
        assert itg == ito and cg == co
        assert sg == pytest.approx(so, rel=1e-10)


def test_default_thresholds_termination(oracle):
    X, ys = instance(oracle, "sqnorm-uniform", 1000, 5, 0.1, 1)
    s, _, _ = oracle.sigma_C(X)
    g = gpu_run(X, ys, sigma_C=s)
    o = oracle_run(oracle, X, ys, sigma_C=s)
    assert o.reason == "thresholds"
    assert_parity(g, o)
    # delta estimate and final dual value (papg.cpp:272-275)
    assert g["res"].delta_estimate == pytest.approx(o.delta_estimate, rel=1e-8)


def test_dual_gradient_ascent_parity(oracle):
    X, ys = instance(oracle, "maxaffine-uniform", 500, 10, 0.1, 9, 20)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=120, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    assert_parity(gpu_run(X, ys, momentum=False, **kw), oracle_run(oracle, X, ys, momentum=False, **kw))


def test_ball_binding_adaptive_restarts(oracle):
    """Tiny B_theta: Q2 clips every iterate; loose thresholds stop at once, the
    saturated norm triggers the doubling warm restarts (papg.cpp:238-251)."""
    X, ys = instance(oracle, "sqnorm-uniform", 200, 3, 0.1, 5)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=400, gap_norm_tol=1e9, infeas_norm_tol=1e9, sigma_C=s, B_theta=1e-5)
    g, o = gpu_run(X, ys, **kw), oracle_run(oracle, X, ys, **kw)
    assert o.restarts >= 3
    assert_parity(g, o)
    assert g["res"].B_theta == o.B_theta == pytest.approx(1e-5 * 2 ** o.restarts)
    kw.update(gap_norm_tol=-1.0, infeas_norm_tol=-1.0, max_iters=80, adaptive_B_theta=False)
    assert_parity(gpu_run(X, ys, **kw), oracle_run(oracle, X, ys, **kw))


def test_warm_start_parity(oracle):
    X, ys = instance(oracle, "maxaffine-uniform", 260, 6, 0.1, 12, 8)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=30, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    first = oracle_run(oracle, X, ys, **kw)
    rng = np.random.default_rng(0)
    theta0 = first.theta * 3e4 + rng.normal(size=first.theta.size) * 1e-3  # forces clipping
    kw["B_theta"] = 20.0
    assert_parity(gpu_run(X, ys, theta0=theta0, **kw),
                  oracle_run(oracle, X, ys, theta0=theta0, **kw))


def test_warm_start_wrong_size_rejected(oracle):
    """papg.cpp:160-161: a warm start of the wrong length is an invalid_argument."""
    X, ys = instance(oracle, "sqnorm-uniform", 120, 3, 0.1, 3)
    with crb.DualSolver(X, ys) as s:
        with pytest.raises(ValueError, match="warm-start"):
            s.begin(crb.PapgConfig(max_iters=2, sigma_C=10.0), True, np.zeros(120 * 119))


def test_theta_row_windows_match_full_export(oracle):
    """cr_get_theta_rows / cr_get_rows_window (spot checks at cfg 5 sizes) are
    slices of the full exports."""
    X, ys = instance(oracle, "maxaffine-uniform", 333, 7, 0.1, 21, 5)
    with crb.DualSolver(X, ys) as s:
        s.begin(crb.PapgConfig(max_iters=9, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=50.0))
        s.iterate(100)
        th, ce = s.theta(), s.rows()
        N = 333
        for a, b in ((0, 1), (5, 77), (300, 333), (0, 333), (17, 17)):
            w = s.theta_rows(a, b)
            assert np.array_equal(w[: (b - a) * (N - 1)], th[a * (N - 1):b * (N - 1)])
            assert np.array_equal(w[(b - a) * (N - 1):], th[N * (N - 1):])
            r = s.rows_window(a, b)
            assert np.array_equal(r[: (b - a) * (N - 1)], ce[a * (N - 1):b * (N - 1)])
            assert np.array_equal(r[(b - a) * (N - 1):], ce[N * (N - 1):])
        with pytest.raises(ValueError):
            s.theta_rows(10, 400)


def test_graph_and_direct_modes_bitwise_identical(oracle):
    X, ys = instance(oracle, "sqnorm-uniform", 700, 5, 0.1, 4)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=150, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    a = gpu_run(X, ys, graph_iters=16, **kw)
    b = gpu_run(X, ys, graph_iters=-1, **kw)
    c = gpu_run(X, ys, graph_iters=-1, **kw)
    assert np.array_equal(a["theta"], b["theta"]) and np.array_equal(a["y"], b["y"])
    assert np.array_equal(b["theta"], c["theta"])  # run-to-run determinism


def test_iterate_in_pieces_matches_one_call(oracle):
    X, ys = instance(oracle, "sqnorm-uniform", 500, 4, 0.1, 8)
    s, _, _ = oracle.sigma_C(X)
    cfg = crb.PapgConfig(max_iters=97, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    with crb.DualSolver(X, ys) as d:
        d.begin(cfg)
        done = 0
        for k in (1, 2, 7, 30, 100):
            done, stopped = d.iterate(k)
        assert done == 97 and stopped
        piecewise = d.theta()
    whole = gpu_run(X, ys, max_iters=97, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    assert np.array_equal(piecewise, whole["theta"])


def test_row_sharded_emulation_on_one_gpu(oracle):
    """Two handles own row blocks [0, N/2) and [N/2, N) of the pair matrix; the
    per-iteration aggregate exchange (the NCCL allreduce payload) is summed on
    the host. The sharded iterates must match the unsharded ones."""
    X, ys = instance(oracle, "maxaffine-uniform", 420, 10, 0.1, 21, 20)
    s, _, _ = oracle.sigma_C(X)
    N = X.shape[0]
    cfg = crb.PapgConfig(max_iters=40, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    cut = 173
    shards = [crb.DualSolver(X, ys, row_begin=0, row_end=cut),
              crb.DualSolver(X, ys, row_begin=cut, row_end=N)]
    try:
        for d in shards:
            d.begin(cfg)
        for _ in range(40):
            for d in shards:
                d.iter_local()
            total = shards[0].exchange_get() + shards[1].exchange_get()
            for d in shards:
                d.exchange_put(total)
            stops = [d.iter_finish() for d in shards]
            assert stops[0] == stops[1]
        th = [d.theta() for d in shards]
        theta = np.concatenate([th[0][: cut * (N - 1)], th[1][: (N - cut) * (N - 1)], th[0][-N:]])
        res = [d.finish() for d in shards]
    finally:
        for d in shards:
            d.close()
    o = oracle_run(oracle, X, ys, max_iters=40, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    assert rel(theta, o.theta) <= TOL_THETA
    assert rel(res[0][1], o.y) <= TOL_Y and np.array_equal(res[0][1], res[1][1])


def test_sharded_time_budget_is_rank_consistent(oracle):
    """Shards whose clocks disagree (the second begins 0.15 s after the first)
    still stop on the same iteration for the time budget: every rank tests the
    budget against the clock slot of the summed payload, which carries the
    elapsed time of the shard owning row 0 (papg.cpp:233-236). A rank that
    stopped on its own clock would leave the others blocked in the next
    allreduce."""
    import time

    X, ys = instance(oracle, "maxaffine-uniform", 300, 5, 0.1, 3, 10)
    N, cut = X.shape[0], 140
    cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=50.0,
                         max_seconds=0.4)
    shards = [crb.DualSolver(X, ys, row_begin=0, row_end=cut),
              crb.DualSolver(X, ys, row_begin=cut, row_end=N)]
    try:
        shards[0].begin(cfg)
        time.sleep(0.15)
        shards[1].begin(cfg)
        for it in range(100000):
            for d in shards:
                d.iter_local()
            total = shards[0].exchange_get() + shards[1].exchange_get()
            for d in shards:
                d.exchange_put(total)
            stops = [d.iter_finish() for d in shards]
            assert stops[0] == stops[1], it
            if stops[0]:
                break
        res = [d.finish()[0] for d in shards]
    finally:
        for d in shards:
            d.close()
    assert res[0].iters == res[1].iters
    assert res[0].reason == res[1].reason == 2  # time budget


def test_nonfinite_gradient_raises():
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, size=(50, 3))
    ys = rng.uniform(1, 2, size=50)
    ys[7] = 1e308  # rows overflow to inf
    with pytest.raises(RuntimeError, match="non-finite"):
        gpu_run(X, ys, max_iters=5, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=50.0)


def test_iterate_before_begin_raises():
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, size=(20, 2))
    with crb.DualSolver(X, np.ones(20)) as d:
        with pytest.raises((ValueError, RuntimeError)):
            d.iterate(1)  # before begin


def _numpy_primal(theta, X, ys, gamma, N):
    th = theta[: N * (N - 1)].reshape(N, N - 1)
    full = np.zeros((N, N))
    mask = ~np.eye(N, dtype=bool)
    full[mask] = th.reshape(-1)
    rows, cols = full.sum(1), full.sum(0)
    y = ys + theta[N * (N - 1):] + rows - cols
    xi = (cols[:, None] * X - full.T @ X) / gamma
    return y, xi


@pytest.mark.parametrize("kind,N,n,noise,pieces,iters", [
    ("maxaffine-uniform", 10000, 10, 0.1, 20, 25),   # BASELINE config 2
    ("lse-uniform", 20000, 20, 0.05, 50, 10),        # BASELINE config 3
])
def test_full_size_properties(kind, N, n, noise, pieces, iters):
    """At BASELINE sizes the oracle is too slow; size-independent properties:
    theta in Q2, diagonal-free, the returned primal equals the closed form of
    the exported theta (aggregation identity), history consistent."""
    d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, noise, 1, pieces))
    p = crb.prepare_problem(d)
    g = gpu_run(p.data.xs, p.data.ys, max_iters=iters, gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
    th = g["theta"]
    assert th.min() >= 0.0
    assert np.linalg.norm(th) <= g["res"].B_theta * (1 + 1e-12)
    y, xi = _numpy_primal(th, p.data.xs, p.data.ys, 1e-3, N)
    assert rel(g["y"], y) <= 1e-10
    assert rel(g["xi"], xi.reshape(-1)) <= 1e-9
    h = g["hist"]
    assert h.shape[0] == iters and np.all(np.isfinite(h))
    assert np.all(np.diff(h[:, 0]) == 1)
    # infeasibility of the last eta from the exported rows
    r = g["rows"]
    infeas = np.linalg.norm(np.minimum(r[: N * (N - 1)], 0))
    assert infeas == pytest.approx(h[-1, 3], rel=1e-9)


def _demo_input(oracle, tmp_path, X, y, iters, sigma, K, mode):
    P = oracle.prepare(X, y)
    inp = tmp_path / f"in{K}_{mode}.bin"
    np.concatenate([[X.shape[0], X.shape[1], iters, sigma, K, mode], X.reshape(-1), P.ys,
                    P.feas_y, P.feas_xi, [P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma]]
                   ).astype(np.float64).tofile(inp)
    return P, inp


def _run_demo(inp, tmp_path):
    exe = os.path.join(ROOT, "paper_1407_7220_b200", "cxx_dropin_demo")
    assert os.path.exists(exe), "built by __graft_entry__.build()"
    out = tmp_path / "out.bin"
    subprocess.run([exe, str(inp), str(out)], check=True)
    return np.fromfile(out, dtype=np.float64)


def test_cpp_dropin_binary(oracle, tmp_path):
    X, y = oracle.gen_instance("maxaffine-uniform", 240, 5, 0.1, 3, 8)
    s, _, _ = oracle.sigma_C(X)
    P, inp = _demo_input(oracle, tmp_path, X, y, 50, s, 0, 0)
    res = _run_demo(inp, tmp_path)
    N = X.shape[0]
    iters, yy, theta = int(res[0]), res[1:1 + N], res[1 + N:]
    o = oracle_run(oracle, X, P.ys, max_iters=50, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                   sigma_C=s)
    assert iters == o.iters
    assert rel(theta, o.theta) <= TOL_THETA and rel(yy, o.y) <= TOL_Y


def test_cpp_dropin_general_k_and_alcc(oracle, tmp_path):
    """papg_solve with a K-block partition and alcc_solve through the C++ drop-in"""
    X, y = oracle.gen_instance("sqnorm-uniform", 36, 2, 0.2, 5)
    K = 3
    s = oracle.sigma_C_k(X, K)[0]
    P, inp = _demo_input(oracle, tmp_path, X, y, 3, s, K, 0)
    res = _run_demo(inp, tmp_path)
    N = 36
    o = oracle.papg_k(X, P.ys, K, P.feas_y, P.feas_xi, inner=dict(max_outer=6, mapg_cap=1000),
                      sigma_C=s, max_iters=3, gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
    assert int(res[0]) == o.iters
    assert rel(res[1 + N:], o.theta) <= 1e-9 and rel(res[1:1 + N], o.y) <= 1e-8
    P, inp = _demo_input(oracle, tmp_path, X, y, 4, 0.0, 0, 1)
    res = _run_demo(inp, tmp_path)
    oa = oracle.alcc(X, P.ys, gamma=P.gamma, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi,
                     warm_y=P.feas_y, warm_xi=P.feas_xi, max_outer=4, mapg_cap=1000,
                     want_multiplier=True)
    assert int(res[0]) == oa.outer_iters
    assert rel(res[1:1 + N], oa.y) <= 1e-9
    assert rel(res[1 + N:], oa.multiplier) <= 1e-6


def test_nccl_attached_single_rank(oracle):
    """The NCCL exchange path (in-graph allreduce + separate control launch) with
    a one-rank communicator reproduces the unsharded iterates."""
    X, ys = instance(oracle, "maxaffine-uniform", 300, 7, 0.1, 31, 9)
    s, _, _ = oracle.sigma_C(X)
    o = oracle_run(oracle, X, ys, max_iters=50, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    for graph_iters in (8, -1):
        cfg = crb.PapgConfig(max_iters=50, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s,
                             graph_iters=graph_iters)
        with crb.DualSolver(X, ys) as d:
            d.attach_nccl(crb.DualSolver.nccl_unique_id(), 0, 1)
            d.begin(cfg)
            done, stopped = d.iterate(1 << 30)
            assert done == 50 and stopped
            res, y, xi, hist = d.finish()
            assert rel(d.theta(), o.theta) <= TOL_THETA
            assert rel(y, o.y) <= TOL_Y


def test_metric_sweeps_match_oracle(oracle):
    """f3: infeasibility, duality gap, estimator and repair (metrics.cpp:8-56)."""
    X, ys = instance(oracle, "maxaffine-uniform", 347, 6, 0.1, 41, 7)
    s, _, _ = oracle.sigma_C(X)
    o = oracle_run(oracle, X, ys, max_iters=40, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    rng = np.random.default_rng(3)
    with crb.DualSolver(X, ys) as d:
        d.begin(crb.PapgConfig(max_iters=40, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s))
        d.iterate(100)
        res, y, xi, _ = d.finish()
        for (py, pxi) in [(o.y, o.xi.reshape(-1)), (rng.normal(size=347), rng.normal(size=347 * 6))]:
            gi = d.infeasibility(py, pxi)
            oi = oracle.infeasibility(X, py, pxi)
            assert gi[0] == pytest.approx(oi[0], rel=1e-11) and gi[1] == pytest.approx(oi[1], rel=1e-11)
            gg = d.duality_gap(py, pxi)
            og = oracle.duality_gap(X, o.theta, py, pxi)
            assert gg[0] == pytest.approx(og[0], rel=1e-9, abs=1e-12 * abs(og[0]) + 1e-300)
        Xq = rng.uniform(-1.2, 1.2, size=(50, 6))
        est = d.evaluate_estimator(o.y, o.xi, Xq)
        ref = np.array([oracle.evaluate_estimator(X, o.y, o.xi, q) for q in Xq])
        assert np.allclose(est, ref, rtol=1e-13, atol=1e-13)
        rep = d.repair_feasibility(o.y, o.xi)
        assert np.allclose(rep, oracle.repair_feasibility(X, o.y, o.xi), rtol=1e-13, atol=1e-13)
        assert np.all(rep >= o.y - 1e-12)


def test_gamma_continuation_resume(oracle):
    """Device-resident warm start across a gamma stage (runner.cpp:258-259, 305,
    322): stage 2 at gamma/10 from stage 1's theta1 equals the oracle with
    theta0 = stage-1 theta."""
    X, y = oracle.gen_instance("lse-uniform", 240, 5, 0.05, 8, 9)
    p1 = oracle.prepare(X, y, 1e-3)
    p2 = oracle.prepare(X, y, 1e-4)
    s, _, _ = oracle.sigma_C(X)
    kw1 = dict(max_iters=30, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    o1 = oracle_run(oracle, X, p1.ys, gamma=1e-3, **kw1)
    o2 = oracle_run(oracle, X, p2.ys, gamma=1e-4, theta0=o1.theta, B_theta=0.5, **kw1)
    with crb.DualSolver(X, p1.ys) as d:
        d.begin(crb.PapgConfig(gamma=1e-3, **kw1))
        d.iterate(1 << 20)
        d.finish()
        assert rel(d.theta(), o1.theta) <= TOL_THETA
        d.set_observations(p2.ys)
        d.begin_resume(crb.PapgConfig(gamma=1e-4, B_theta=0.5, **kw1))
        done, stopped = d.iterate(1 << 20)
        res, y2, xi2, _ = d.finish()
        assert done == o2.iters
        assert rel(d.theta(), o2.theta) <= TOL_THETA
        assert rel(y2, o2.y) <= TOL_Y


@pytest.mark.parametrize("path", ["small", "mma"])
@pytest.mark.parametrize("N,n", [(2, 1), (3, 2), (17, 16), (21, 20), (25, 24), (33, 5), (65, 13),
                                 (33, 32), (47, 27)])
def test_tiny_and_ragged_sizes(oracle, monkeypatch, path, N, n):
    """Edge sizes: N = n + 1, N below one strip/tile, ragged last strips."""
    monkeypatch.setenv("CRB_SMALL", "1" if path == "small" else "0")
    X, ys = instance(oracle, "sqnorm-uniform", N, n, 0.1, 77)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=25, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    assert_parity(gpu_run(X, ys, **kw), oracle_run(oracle, X, ys, **kw))


@pytest.mark.parametrize("kind,N,n,pieces", [("maxaffine-uniform", 1000, 10, 8),
                                             ("lse-uniform", 777, 20, 12),
                                             ("sqnorm-uniform", 503, 3, 0)])
def test_tensor_map_producer_bitwise_equals_row_copies(oracle, monkeypatch, kind, N, n, pieces):
    """The DMMA P-APG producer loads a stage with one 3-D tensor TMA per buffer
    (pitch padding zero-filled out of bounds); CRB_TMAP=0 keeps the per-row bulk
    copies. Same shared-memory contents -> bitwise identical solves, both at
    oracle parity (ragged N: the last tile's view runs past ld)."""
    monkeypatch.setenv("CRB_SMALL", "0")
    X, ys = instance(oracle, kind, N, n, 0.1, 21, pieces)
    s, _, _ = oracle.sigma_C(X)
    kw = dict(max_iters=120, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, sigma_C=s)
    a = gpu_run(X, ys, **kw)
    monkeypatch.setenv("CRB_TMAP", "0")
    b = gpu_run(X, ys, **kw)
    assert np.array_equal(a["theta"], b["theta"]) and np.array_equal(a["y"], b["y"])
    assert_parity(a, oracle_run(oracle, X, ys, **kw))


def test_alcc_penalty_sweep_tensor_map_bitwise(oracle, monkeypatch):
    """The ALCC penalty sweeps (per-kernel path, CRB_ALCC_LOOP=0) read theta
    through the same tensor map: bitwise identical to the per-row copies."""
    monkeypatch.setenv("CRB_ALCC_LOOP", "0")
    X, y = oracle.gen_instance("maxaffine-uniform", 900, 6, 0.1, 5, 6)
    P = oracle.prepare(X, y, 1e-3)
    cfg = crb.AlccConfig(sigma_A1=oracle.sigma_A(X, 1)[0], sigma_A2=oracle.sigma_A(X, 2)[0],
                         max_outer=2)
    bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma)
    out = []
    for tm in ("1", "0"):
        monkeypatch.setenv("CRB_TMAP", tm)
        with crb.DualSolver(X, P.ys, P.gamma) as s:
            res, yy, xi, hist, mi = s.alcc(cfg, bounds, crb.PrimalPoint(P.feas_y, P.feas_xi))
            out.append((res.outer_iters, list(mi), yy, xi, s.alcc_multiplier()))
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    for k in (2, 3, 4):
        assert np.array_equal(out[0][k], out[1][k])


@pytest.mark.parametrize("grid", ["148", "64", "7"])
def test_sigma_power_grid_sizes(oracle, monkeypatch, grid):
    """One-barrier power loop: same step count and sigma (1e-10) for any grid."""
    X, _ = instance(oracle, "maxaffine-uniform", 3000, 8, 0.1, 9, 10)
    so, it_o, _ = oracle.sigma_C(X)
    monkeypatch.setenv("CRB_POWER_GRID", grid)
    with crb.DualSolver(X, np.zeros(len(X))) as d:
        sg, it_g, conv = d.sigma_C()
    assert it_g == it_o and conv
    assert abs(sg - so) <= 1e-10 * so


@pytest.mark.parametrize("path", ["cluster", "grid"])
@pytest.mark.parametrize("kind,N,n,pieces", [("maxaffine-uniform", 2100, 10, 20),
                                             ("sqnorm-uniform", 1777, 5, 0),
                                             ("quadratic", 901, 1, 0)])
def test_sigma_cluster_and_grid_paths(oracle, monkeypatch, path, kind, N, n, pieces):
    """sigma_max(C) from the single-cluster power loop (DSMEM records, n <= 10)
    and from the cooperative grid loop: the oracle's step count and sigma."""
    if path == "grid":
        monkeypatch.setenv("CRB_SIGMA_CLUSTER", "0")
    X, _ = instance(oracle, kind, N, n, 0.1, 5, pieces)
    so, it_o, co = oracle.sigma_C(X)
    with crb.DualSolver(X, np.zeros(len(X))) as d:
        sg, it_g, cg = d.sigma_C()
    assert it_g == it_o and cg == co
    assert abs(sg - so) <= 1e-10 * so

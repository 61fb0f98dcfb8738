"""Pins the memory-light replay oracle (cro_papg_replay) to the literal oracle.

cro_papg_replay restates the same loop (papg.cpp:136-283) without any N^2
array: it keeps the per-iteration primal and step scalars and recomputes each
pair's multiplier history on every pass. It is the checker for BASELINE
configs 4 and 5, whose dual vectors (2.5e9 / 1e10 pairs per copy) do not fit
a literal run's four N^2 arrays on the host. With one thread it must be
bitwise equal to the literal oracle; with several it differs only in the
association of the per-thread sums.
"""
import numpy as np
import pytest


def _inst(oracle, kind, N, n, noise, seed, pieces=0):
    X, y = oracle.gen_instance(kind, N, n, noise, seed, pieces)
    p = oracle.prepare(X, y)
    s, _, _ = oracle.sigma_C(X)
    return X, p.ys, s


def _rows(theta, N, rows):
    return np.concatenate([theta[r * (N - 1):(r + 1) * (N - 1)] for r in rows] +
                          [theta[N * (N - 1):]])


CASES = {
    "fixed_iters": dict(max_iters=40, gap_norm_tol=-1.0, infeas_norm_tol=-1.0),
    "thresholds": dict(max_iters=500),
    "dga": dict(max_iters=30, use_momentum=False, gap_norm_tol=-1.0, infeas_norm_tol=-1.0),
    "ball_restarts": dict(max_iters=400, gap_norm_tol=1e9, infeas_norm_tol=1e9, B_theta=1e-5),
    "ball_fixed": dict(max_iters=25, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, B_theta=1e-5,
                       adaptive_B_theta=False),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_replay_bitwise_single_thread(oracle, case):
    kind, N, n = ("sqnorm-uniform", 60, 3) if "ball" in case else ("maxaffine-uniform", 70, 4)
    X, ys, s = _inst(oracle, kind, N, n, 0.1, 5, 6)
    kw = dict(CASES[case], sigma_C=s)
    a = oracle.papg(X, ys, want_c_eta=True, **kw)
    b = oracle.papg_replay(X, ys, rows=range(N), **kw)
    if case == "ball_restarts":
        assert a.restarts >= 3
    assert (a.iters, a.reason, a.restarts, a.saturated) == (b.iters, b.reason, b.restarts, b.saturated)
    assert np.array_equal(a.theta, b.theta)
    assert np.array_equal(a.c_eta, b.c_eta)
    assert np.array_equal(a.y, b.y) and np.array_equal(a.xi, b.xi)
    assert np.array_equal(a.history[:, 1:7], b.history[:, 1:7])
    assert a.g_final == b.g_final and a.delta_estimate == b.delta_estimate
    assert a.B_theta == b.B_theta


@pytest.mark.parametrize("case", ["fixed_iters", "ball_restarts", "dga"])
def test_replay_threads_and_row_window(oracle, case):
    kind, N, n = ("sqnorm-uniform", 60, 3) if "ball" in case else ("maxaffine-uniform", 90, 5)
    X, ys, s = _inst(oracle, kind, N, n, 0.1, 8, 7)
    kw = dict(CASES[case], sigma_C=s)
    a = oracle.papg(X, ys, want_c_eta=True, **kw)
    rows = [0, 3, 13, 14, 15, 40, N - 1]
    b = oracle.papg_replay(X, ys, rows=rows, threads=4, **kw)
    assert (a.iters, a.reason, a.restarts) == (b.iters, b.reason, b.restarts)
    for ref, got in ((a.theta, b.theta), (a.c_eta, b.c_eta)):
        ref = _rows(ref, N, rows)
        assert np.linalg.norm(got - ref) <= 1e-14 * np.linalg.norm(ref)
    assert np.linalg.norm(b.y - a.y) <= 1e-14 * np.linalg.norm(a.y)
    assert np.allclose(b.history[:, 1:7], a.history[:, 1:7], rtol=1e-12, atol=1e-14)

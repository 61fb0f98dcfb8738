"""Pins the oracle's standalone ALCC restatement (oracle/cvxreg_oracle.c:
cro_alcc, cro_sigma_A) against an independent dense numpy restatement of the
same reference text (alcc.cpp:54-208, engines.cpp:57-106, operators.cpp:302-351,
projections.hpp:22-26). CPU only."""
import numpy as np
import pytest

from oracle import oracle as O


def dense_rows(X):
    """A = [A1 | A2] over the canonical (l1, l2 != l1) rows: y_l1 - y_l2 - xi_l2.(x_l1 - x_l2)."""
    N, n = X.shape
    m = N * (N - 1)
    A = np.zeros((m, N + N * n))
    r = 0
    for l1 in range(N):
        for l2 in range(N):
            if l1 == l2:
                continue
            A[r, l1] += 1.0
            A[r, l2] -= 1.0
            A[r, N + l2 * n: N + (l2 + 1) * n] = -(X[l1] - X[l2])
            r += 1
    return A


def power_sigma(M, tol=1e-6, max_iters=5000):
    """operators.cpp:302-339 with a numpy operator and the reference's seeded start."""
    v = O.rng_draws(0x5EED, 97, M.shape[1], "normal")
    v = v / np.linalg.norm(v)
    lam_prev = 0.0
    for it in range(1, max_iters + 1):
        w = M @ v
        lam = w @ w
        u = M.T @ w
        nu = np.linalg.norm(u)
        v = u / nu
        if it > 1 and abs(lam - lam_prev) <= tol * lam:
            return np.sqrt(lam) * 1.01, it
        lam_prev = lam
    return np.sqrt(lam_prev) * 1.10, max_iters


def project_ball(v, c, r):
    d = np.linalg.norm(v - c)
    return c + (r / d) * (v - c) if d > r else v


def dense_alcc(X, ys, gamma, By, Bx, sA1, sA2, wy, wxi, mu1=1.0, tau1=1e-2, alpha1=1e-3, c=5.0,
               kappa=0.5, max_outer=30, cap=200000, itol=1e-1, gtol=1e-6):
    N, n = X.shape
    A = dense_rows(X)
    A1, A2 = A[:, :N], A[:, N:]
    m = A.shape[0]
    cy, cx = ys, np.zeros(N * n)
    theta = np.zeros(m)
    mu = mu1
    y = project_ball(wy.copy(), cy, By)
    xi = project_ball(wxi.copy(), cx, Bx)

    def grad(y, xi):
        res = A1 @ y + A2 @ xi - theta
        v = np.maximum(-res, 0.0)
        return (y - cy) / mu - A1.T @ v, (gamma / mu) * (xi - cx) - A2.T @ v, v

    _, _, v = grad(y, xi)
    p1 = np.sum((y - cy) ** 2) / (2 * mu) + gamma * np.sum(xi ** 2) / (2 * mu) + 0.5 * v @ v
    tau = max(tau1 * p1, 1e-16)
    ay_ = ax_ = alpha1 * (By + Bx)
    out = dict(mapg=[], hist=[])
    for k in range(1, max_outer + 1):
        Ly = 1 / mu + sA1 ** 2
        Lx = gamma / mu + sA2 ** 2
        lmax = int(np.ceil(4 * np.sqrt((Ly * By ** 2 + Lx * Bx ** 2) / tau)))
        lmax = min(max(lmax, 10), cap)
        y1p, y1, y2 = y.copy(), y.copy(), y.copy()
        x1p, x1, x2 = xi.copy(), xi.copy(), xi.copy()
        t = 1.0
        inner = 0
        for ell in range(1, lmax + 1):
            gy, gx, _ = grad(y2, x2)
            y1p, y1 = y1, project_ball(y2 - gy / Ly, cy, By)
            x1p, x1 = x1, project_ball(x2 - gx / Lx, cx, Bx)
            inner = ell
            dy, dx = np.linalg.norm(y1 - y2), np.linalg.norm(x1 - x2)
            tn = 0.5 * (1 + np.sqrt(1 + 4 * t * t))
            y2 = y1 + ((t - 1) / tn) * (y1 - y1p)
            x2 = x1 + ((t - 1) / tn) * (x1 - x1p)
            t = tn
            if dy <= ay_ and dx <= ax_:
                break
        y, xi = y1, x1
        out["mapg"].append(inner)
        res = A1 @ y + A2 @ xi
        vneg = np.maximum(theta - res, 0.0)
        lam = mu * vneg
        infeas = np.linalg.norm(np.maximum(-res, 0.0))
        gap = lam @ res
        adj_y, adj_x = A1.T @ lam, A2.T @ lam
        dual = -0.5 * adj_y @ adj_y - adj_x @ adj_x / (2 * gamma) - lam @ (A1 @ cy)
        primal = 0.5 * np.sum((y - cy) ** 2) + 0.5 * gamma * np.sum(xi ** 2)
        out["hist"].append((k, infeas, gap, primal - dual))
        out.update(y=y, xi=xi, lam=lam, certified=primal - dual, k=k)
        if infeas / np.sqrt(m) <= itol and abs(gap / m) <= gtol:
            out["reason"] = "thresholds"
            return out
        theta = vneg / c
        mu *= c
        decay = (c * k ** (1 + kappa)) ** 2
        tau /= decay
        ay_ /= decay
        ax_ /= decay
    out["reason"] = "iter_budget"
    return out


@pytest.mark.parametrize("N,n,seed", [(7, 1, 1), (9, 2, 2), (8, 3, 5)])
def test_sigma_A_matches_dense(N, n, seed):
    X, _ = O.gen_instance("sqnorm-uniform", N, n, noise=0.1, seed=seed)
    A = dense_rows(X)
    for which, M in ((1, A[:, :N]), (2, A[:, N:])):
        s, it, cv = O.sigma_A(X, which)
        s_ref, it_ref = power_sigma(M)
        assert cv and it == it_ref
        assert s == pytest.approx(s_ref, rel=1e-12)
        # and the estimate is the spectral norm inflated by 1.01 (operators.cpp:334)
        assert s / 1.01 == pytest.approx(np.linalg.norm(M, 2), rel=1e-5)
    # A1^T A1 = 2 (N I - 1 1^T): sigma_max(A1) = sqrt(2N)
    assert O.sigma_A(X, 1)[0] == pytest.approx(1.01 * np.sqrt(2 * N), rel=1e-12)


@pytest.mark.parametrize("N,n,seed,max_outer", [(8, 1, 3, 6), (10, 2, 4, 8), (9, 3, 7, 5)])
def test_alcc_matches_dense_restatement(N, n, seed, max_outer):
    X, y = O.gen_instance("sqnorm-uniform", N, n, noise=0.3, seed=seed)
    P = O.prepare(X, y, 1e-3)
    s1, s2 = O.sigma_A(X, 1)[0], O.sigma_A(X, 2)[0]
    kw = dict(gamma=1e-3, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, sigma_A1=s1, sigma_A2=s2,
              max_outer=max_outer, mapg_cap=3000)
    r = O.alcc(X, P.ys, warm_y=P.feas_y, warm_xi=P.feas_xi, want_multiplier=True, **kw)
    d = dense_alcc(X, P.ys, 1e-3, P.Bbar_y, P.Bbar_xi, s1, s2, P.feas_y, P.feas_xi,
                   max_outer=max_outer, cap=3000)
    assert r.outer_iters == d["k"]
    assert r.reason == d["reason"]
    assert list(r.mapg_iters) == d["mapg"]
    scale = max(1.0, np.abs(d["y"]).max())
    assert np.abs(r.y - d["y"]).max() <= 1e-9 * scale
    assert np.abs(r.xi.reshape(-1) - d["xi"]).max() <= 1e-9 * max(1.0, np.abs(d["xi"]).max())
    assert np.abs(r.multiplier - d["lam"]).max() <= 1e-9 * max(1.0, np.abs(d["lam"]).max())
    for h, (k, inf, gap, cert) in zip(r.history, d["hist"]):
        assert h[0] == k
        assert h[3] == pytest.approx(inf, rel=1e-9, abs=1e-12)
        assert h[5] == pytest.approx(gap, rel=1e-8, abs=1e-12)
    assert r.certified_gap == pytest.approx(d["certified"], rel=1e-8, abs=1e-10)


def test_alcc_invalid_config():
    X, y = O.gen_instance("sqnorm-uniform", 6, 1, noise=0.1, seed=1)
    P = O.prepare(X, y, 1e-3)
    base = dict(gamma=1e-3, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, warm_y=P.feas_y,
                warm_xi=P.feas_xi)
    for bad in (dict(c=1.0), dict(kappa=0.0), dict(mu1=0.0)):  # alcc.cpp:59-61
        with pytest.raises(RuntimeError):
            O.alcc(X, P.ys, **base, **bad)


def test_alcc_feasible_warm_start_reduces_objective():
    """The ALCC from the feasible affine slice approaches the LSE fit: the
    objective drops well below the affine fit's and the rows end near-feasible."""
    X, y = O.gen_instance("sqnorm-uniform", 30, 2, noise=0.05, seed=11)
    P = O.prepare(X, y, 1e-3)
    r = O.alcc(X, P.ys, gamma=1e-3, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, warm_y=P.feas_y,
               warm_xi=P.feas_xi, max_outer=12, infeas_norm_tol=1e-4, gap_norm_tol=1e-8)
    affine = 0.5 * np.sum((P.feas_y - P.ys) ** 2)
    assert r.objective < 0.5 * affine
    raw, norm = O.infeasibility(X, r.y, r.xi)
    assert norm < 1e-3

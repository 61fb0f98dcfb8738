"""Pins the oracle's general-K P-APG(ALCC) restatement (cro_papg_k,
cro_apply_C_k, cro_sigma_C_k) against an independent dense numpy restatement
of the same reference text: the cross-block operator C (operators.cpp:128-180,
indexing.hpp:9-37), the block QPs (alcc_solve_block alcc.cpp:222-258 on the
within rows, alcc_core :54-191 with the target_subopt stop) and the dual loop
(papg.cpp:136-283). CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from test_alcc_oracle import dense_rows, power_sigma, project_ball


def dense_C(X, K):
    N, n = X.shape
    nb = N // K
    rows = []
    for i in range(K):
        for j in range(K):
            if i == j:
                continue
            for l1 in range(i * nb, (i + 1) * nb):
                for l2 in range(j * nb, (j + 1) * nb):
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


def dense_block_alcc(Xb, cy, cx, gamma, By, Bx, s1, s2, wy, wx, target, cfg):
    """alcc_core on the within rows of one block with centres (cy, cx)."""
    nb, n = Xb.shape
    A = dense_rows(Xb)
    A1, A2 = A[:, :nb], A[:, nb:]
    m = A.shape[0]
    theta = np.zeros(m)
    mu = cfg["mu1"]
    y = project_ball(wy.copy(), cy, By)
    xi = project_ball(wx.copy(), cx, Bx)

    def grad(y, xi):
        res = A1 @ y + A2 @ xi - theta
        v = np.maximum(-res, 0.0)
        return (y - cy) / mu - A1.T @ v, (gamma / mu) * (xi - cx) - A2.T @ v, v

    _, _, v = grad(y, xi)
    p1 = np.sum((y - cy) ** 2) / (2 * mu) + gamma * np.sum((xi - cx) ** 2) / (2 * mu) + 0.5 * v @ v
    tau = max(cfg["tau1_scale"] * p1, 1e-16)
    ay_ = ax_ = cfg["alpha1_scale"] * (By + Bx)
    rows_center = A1 @ cy + A2 @ cx
    iters = 0
    infeas = 0.0
    for k in range(1, cfg["max_outer"] + 1):
        Ly = 1 / mu + s1 ** 2
        Lx = gamma / mu + s2 ** 2
        lmax = int(np.ceil(4 * np.sqrt((Ly * By ** 2 + Lx * Bx ** 2) / tau)))
        lmax = min(max(lmax, 10), cfg["mapg_cap"])
        y1p, y1, y2 = y.copy(), y.copy(), y.copy()
        x1p, x1, x2 = xi.copy(), xi.copy(), xi.copy()
        t = 1.0
        for ell in range(1, lmax + 1):
            gy, gx, _ = grad(y2, x2)
            y1p, y1 = y1, project_ball(y2 - gy / Ly, cy, By)
            x1p, x1 = x1, project_ball(x2 - gx / Lx, cx, Bx)
            iters += 1
            dy, dx = np.linalg.norm(y1 - y2), np.linalg.norm(x1 - x2)
            tn = 0.5 * (1 + np.sqrt(1 + 4 * t * t))
            y2 = y1 + ((t - 1) / tn) * (y1 - y1p)
            x2 = x1 + ((t - 1) / tn) * (x1 - x1p)
            t = tn
            if dy <= ay_ and dx <= ax_:
                break
        y, xi = y1, x1
        res = A1 @ y + A2 @ xi
        vneg = np.maximum(theta - res, 0.0)
        lam = mu * vneg
        infeas = np.linalg.norm(np.maximum(-res, 0.0))
        adj_y, adj_x = A1.T @ lam, A2.T @ lam
        dual = -0.5 * adj_y @ adj_y - adj_x @ adj_x / (2 * gamma) - lam @ rows_center
        primal = 0.5 * np.sum((y - cy) ** 2) + 0.5 * gamma * np.sum((xi - cx) ** 2)
        if primal - dual <= target and np.linalg.norm(lam) * infeas <= target:
            break
        theta = vneg / cfg["c"]
        mu *= cfg["c"]
        decay = (cfg["c"] * k ** (1 + cfg["kappa"])) ** 2
        tau /= decay
        ay_ /= decay
        ax_ /= decay
    return y, xi, infeas, iters


def dense_papg_k(X, ys, K, fy, fx, gamma, sigma_C, max_iters, inner):
    N, n = X.shape
    nb = N // K
    C = dense_C(X, K)
    cross = N * (N - nb)
    L = sigma_C ** 2 / gamma
    s1 = O.sigma_A(X[:nb], 1)[0]
    s2 = [O.sigma_A(X[b * nb:(b + 1) * nb], 2)[0] for b in range(K)]
    warm_y, warm_x = fy.copy(), fx.copy()
    B = 10 * np.sqrt(N)
    th1 = np.zeros(C.shape[0])
    th1p, th2 = th1.copy(), th1.copy()
    t = 1.0
    inner_total = 0

    def dual_grad(theta, tol):
        nonlocal inner_total
        q = C.T @ theta
        qy, qx = q[:N], q[N:]
        ey, ex = np.empty(N), np.empty(N * n)
        for b in range(K):
            sl, sx = slice(b * nb, (b + 1) * nb), slice(b * nb * n, (b + 1) * nb * n)
            cy = ys[sl] + qy[sl]
            cx = qx[sx] / gamma
            Bb = max(np.sqrt(np.sum((fy[sl] - cy) ** 2) + gamma * np.sum((fx[sx] - cx) ** 2)), 1e-8)
            y, xi, _, it = dense_block_alcc(X[sl], cy, cx, gamma, Bb, Bb / np.sqrt(gamma), s1,
                                            s2[b], warm_y[sl], warm_x[sx], tol, inner)
            inner_total += it
            ey[sl], ex[sx] = y, xi
            warm_y[sl], warm_x[sx] = y, xi
        return ey, ex, C @ np.concatenate([ey, ex])

    for ell in range(1, max_iters + 1):
        tol = min(1e-6, 1.0 / ell ** 3)
        ey, ex, ceta = dual_grad(th2, tol)
        th1p, th1 = th1, th2 - ceta / L
        th1 = np.maximum(th1, 0.0)
        nrm = np.linalg.norm(th1)
        if nrm > B:
            th1 *= B / nrm
        tn = 0.5 * (1 + np.sqrt(1 + 4 * t * t))
        th2 = th1 + ((t - 1) / tn) * (th1 - th1p)
        t = tn
    ft = min(1e-10, 1e-6, 1.0 / max_iters ** 3)
    ey, ex, _ = dual_grad(th1, ft)
    return th1, ey, ex, ceta, inner_total, cross


@pytest.mark.parametrize("N,n,K,seed", [(8, 1, 2, 1), (9, 2, 3, 2), (12, 1, 4, 3)])
def test_apply_C_k_and_sigma_match_dense(N, n, K, seed):
    X, _ = O.gen_instance("sqnorm-uniform", N, n, 0.1, seed)
    C = dense_C(X, K)
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(N + N * n)
    np.testing.assert_allclose(O.apply_C_k(X, K, v[:N], v[N:]), C @ v, rtol=1e-13, atol=1e-13)
    w = rng.standard_normal(C.shape[0])
    oy, ox = O.apply_C_T_k(X, K, w)
    np.testing.assert_allclose(np.concatenate([oy, ox]), C.T @ w, rtol=1e-12, atol=1e-12)
    s, it, cv = O.sigma_C_k(X, K)
    s_ref, it_ref = power_sigma(C)
    assert it == it_ref and s == pytest.approx(s_ref, rel=1e-12)
    # K = N falls back to the singleton operator
    assert O.sigma_C_k(X, N)[0] == O.sigma_C(X)[0]


@pytest.mark.parametrize("N,n,K,seed", [(8, 1, 2, 1), (9, 2, 3, 2)])
def test_papg_k_matches_dense_restatement(N, n, K, seed):
    X, y = O.gen_instance("sqnorm-uniform", N, n, 0.2, seed)
    P = O.prepare(X, y, 1e-3)
    inner = dict(O.INNER_DEFAULTS, max_outer=6, mapg_cap=800)
    sig = O.sigma_C_k(X, K)[0]
    o = O.papg_k(X, P.ys, K, P.feas_y, P.feas_xi, inner=inner, sigma_C=sig, max_iters=3,
                 gap_norm_tol=-1.0, want_c_eta=True)
    th, ey, ex, ceta, it, cross = dense_papg_k(X, P.ys, K, P.feas_y, P.feas_xi, 1e-3, sig, 3,
                                               inner)
    assert o.iters == 3
    assert o.extra["inner_iters"] == it
    np.testing.assert_allclose(o.theta, th, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(o.y, ey, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(o.xi.reshape(-1), ex, rtol=1e-8, atol=1e-10)

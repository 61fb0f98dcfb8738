"""Randomised parity sweep of the widening rows against the REFERENCE's own compiled code:
general-K P-APG(ALCC) (f2: papg_solve with K < N blocks) and the standalone ALCC (f1).

    python scripts/fuzz_widening_vs_reference.py [cases] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1407_7220_b200 as crb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

KINDS = [("sqnorm-uniform", 0), ("maxaffine-uniform", 6), ("quadratic", 0), ("exponential", 0)]


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a).ravel() - np.asarray(b).ravel()) / (nb if nb > 0 else 1.0)


def general_case(rng, k):
    kind, pieces = KINDS[rng.integers(len(KINDS))]
    n = int(rng.choice([1, 2, 3, 4, 6]))
    K = int(rng.choice([2, 3, 4, 5, 8]))
    nbar = int(rng.integers(n + 1, 40))
    N = K * nbar
    iters = int(rng.integers(2, 10))
    inner = dict(max_outer=int(rng.integers(3, 9)), mapg_cap=int(rng.choice([300, 800, 1500])))
    X, y = O.gen_instance(kind, N, n, float(rng.uniform(0.1, 0.5)), int(rng.integers(1, 10**6)), pieces)
    P = R.prepare(X, y)
    r = R.papg(X, P.ys, K=K, feas_y=P.feas_y, feas_xi=P.feas_xi, inner=inner, max_iters=iters,
               gap_norm_tol=-1.0, infeas_norm_tol=-1.0, threads=os.cpu_count() or 1)
    cfg = crb.PapgConfig(max_iters=iters, sigma_C=r.sigma_C, K=K, gap_norm_tol=-1.0,
                         infeas_norm_tol=-1.0, inner=crb.AlccConfig(**inner))
    with crb.DualSolver(X, P.ys) as s:
        s.set_partition(K, crb.PrimalPoint(P.feas_y, P.feas_xi), cfg.inner)
        s.begin(cfg, True)
        stopped = False
        while not stopped:
            _, stopped = s.iterate(1 << 40)
        res, yg, xig, hist = s.finish()
        th = s.theta()
    e = rel(th, r.theta), rel(yg, r.y)
    ok = res.iters == r.iters and e[0] <= 1e-9 and e[1] <= 1e-8
    print(f"{k:3d} {'ok ' if ok else 'BAD'} general {kind:18s} N={N:4d} n={n} K={K} nbar={nbar:2d} "
          f"iters={r.iters} inner={inner['max_outer']}/{inner['mapg_cap']} theta {e[0]:.1e} y {e[1]:.1e}",
          flush=True)
    return ok, e


def alcc_case(rng, k):
    kind, pieces = KINDS[rng.integers(len(KINDS))]
    n = int(rng.choice([1, 2, 3, 5, 8]))
    N = int(rng.integers(n + 2, 160))
    mo, cap = int(rng.integers(2, 7)), int(rng.choice([200, 600, 1500]))
    X, y = O.gen_instance(kind, N, n, float(rng.uniform(0.1, 0.5)), int(rng.integers(1, 10**6)), pieces)
    P = R.prepare(X, y)
    s1, s2 = R.sigma(X, "A1"), R.sigma(X, "A2")
    a = R.alcc(X, P.ys, gamma=1e-3, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, warm_y=P.feas_y,
               warm_xi=P.feas_xi, max_outer=mo, mapg_cap=cap)
    cfg = crb.AlccConfig(sigma_A1=s1[0], sigma_A2=s2[0], max_outer=mo, mapg_cap=cap)
    bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, 1e-3)
    with crb.DualSolver(X, P.ys, 1e-3) as s:
        res, yg, xig, hist, mi = s.alcc(cfg, bounds, crb.PrimalPoint(P.feas_y, P.feas_xi))
    same = (res.outer_iters, res.mapg_iters_total, res.reason) == \
        (a.outer_iters, a.mapg_iters_total, O.REASONS_INV[a.reason])
    e = rel(yg, a.y), rel(xig, a.xi)
    # long inner runs amplify last-bit differences with the inner conditioning (test_alcc_gpu.py)
    ok = same and e[0] <= 1e-8 and e[1] <= 1e-7
    print(f"{k:3d} {'ok ' if ok else 'BAD'} alcc    {kind:18s} N={N:4d} n={n} outer={a.outer_iters} "
          f"mapg={a.mapg_iters_total:5d} {a.reason:11s} y {e[0]:.1e} xi {e[1]:.1e}", flush=True)
    return ok, e


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
    bad = 0
    worst = [0.0, 0.0, 0.0, 0.0]
    for k in range(cases):
        ok, e = general_case(rng, k)
        bad += 0 if ok else 1
        worst[0], worst[1] = max(worst[0], e[0]), max(worst[1], e[1])
    for k in range(cases):
        ok, e = alcc_case(rng, k)
        bad += 0 if ok else 1
        worst[2], worst[3] = max(worst[2], e[0]), max(worst[3], e[1])
    print(f"cases {2 * cases}, failures {bad}, worst general (theta, y) = ({worst[0]:.2e}, "
          f"{worst[1]:.2e}), alcc (y, xi) = ({worst[2]:.2e}, {worst[3]:.2e})")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

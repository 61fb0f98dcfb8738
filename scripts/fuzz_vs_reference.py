"""Randomised parity sweep: the CUDA path against the REFERENCE's own compiled code
(oracle/_ref) on many small seeded instances -- sizes around the tile / strip / stage
boundaries, every generator kind, momentum and DGA, binding balls, loose thresholds
(restarts) and both sweep paths. Prints one line per case and the worst errors.

    python scripts/fuzz_vs_reference.py [cases] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1407_7220_b200 as crb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

KINDS = [("sqnorm-uniform", 0), ("maxaffine-uniform", 7), ("lse-uniform", 12), ("quadratic", 0),
         ("exponential", 0)]


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a).ravel() - np.asarray(b).ravel()) / (nb if nb > 0 else 1.0)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
    worst = dict(theta=0.0, y=0.0, xi=0.0, hist=0.0)
    bad = 0
    for k in range(cases):
        kind, pieces = KINDS[rng.integers(len(KINDS))]
        n = int(rng.choice([1, 2, 3, 5, 8, 10, 13, 16, 20, 27, 32]))
        N = int(rng.choice([n + 1, n + 2, 17, 31, 32, 33, 64, 65, 100, 127, 129, 200, 241, 257, 333,
                            400]))
        N = max(N, n + 1)
        iters = int(rng.integers(1, 60))
        mom = bool(rng.integers(0, 4) > 0)
        mode = rng.integers(0, 5)
        kw = dict(gap_norm_tol=-1.0, infeas_norm_tol=-1.0)
        if mode == 0:
            kw = dict(gap_norm_tol=1e9, infeas_norm_tol=1e9, B_theta=10.0 ** rng.uniform(-6, -3))
            iters = 300
        elif mode == 1:
            kw["B_theta"] = 10.0 ** rng.uniform(-4, 0)
        elif mode == 2:
            kw = dict(gap_norm_tol=10.0 ** rng.uniform(-5, -2), infeas_norm_tol=1e-1)
            iters = 4000
        small = str(int(rng.integers(0, 2)))
        os.environ["CRB_SMALL"] = small
        X, y = O.gen_instance(kind, N, n, float(rng.uniform(0.05, 0.5)), int(rng.integers(1, 10**6)),
                              pieces)
        P = R.prepare(X, y)
        r = R.papg(X, P.ys, feas_y=P.feas_y, feas_xi=P.feas_xi, max_iters=iters, use_momentum=mom,
                   **kw)
        cfg = crb.PapgConfig(max_iters=iters, sigma_C=r.sigma_C, **kw)
        with crb.DualSolver(X, P.ys) as s:
            s.begin(cfg, mom)
            stopped = False
            while not stopped:
                _, stopped = s.iterate(1 << 40)
            res, yg, xig, hist = s.finish()
            th = s.theta()
            sg, sit, _ = s.sigma_C()
        same = (res.iters, res.restarts, res.reason, bool(res.saturated)) == \
            (r.iters, r.restarts, O.REASONS_INV[r.reason], r.saturated)
        e = dict(theta=rel(th, r.theta), y=rel(yg, r.y), xi=rel(xig, r.xi))
        scale = np.abs(r.history[:, 1:7]).max(axis=0)
        e["hist"] = float((np.abs(hist[:, 1:7] - r.history[:, 1:7]).max(axis=0) /
                           np.maximum(scale, 1e-300)).max())
        e_sig = abs(sg - r.sigma_C) / r.sigma_C
        ok = same and e["theta"] <= 1e-12 and e["y"] <= 1e-8 and e["hist"] <= 1e-9 and e_sig <= 1e-10
        bad += 0 if ok else 1
        for key in worst:
            worst[key] = max(worst[key], e[key])
        print(f"{k:3d} {'ok ' if ok else 'BAD'} {kind:18s} N={N:4d} n={n:2d} small={small} "
              f"mom={int(mom)} mode={mode} iters={r.iters:4d} restarts={r.restarts} {r.reason:11s} "
              f"theta {e['theta']:.1e} y {e['y']:.1e} xi {e['xi']:.1e} hist {e['hist']:.1e} "
              f"sigma {e_sig:.1e}", flush=True)
    print(f"cases {cases}, failures {bad}, worst {worst}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

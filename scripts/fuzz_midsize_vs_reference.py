"""Mid-size randomised parity sweep against the REFERENCE's own compiled code: ragged N in
[400, 1500] (several column tiles and CTA segments of the DMMA sweep), CRB_SMALL=0.

    python scripts/fuzz_midsize_vs_reference.py [cases] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CRB_SMALL"] = "0"
import paper_1407_7220_b200 as crb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a).ravel() - np.asarray(b).ravel()) / (nb if nb > 0 else 1.0)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
    bad = 0
    worst = [0.0, 0.0]
    for k in range(cases):
        kind, pieces = [("sqnorm-uniform", 0), ("maxaffine-uniform", 12), ("lse-uniform", 20)][rng.integers(3)]
        n = int(rng.choice([2, 5, 7, 10]))
        N = int(rng.integers(400, 1500))
        to_tol = bool(rng.integers(0, 2))
        kw = dict(gap_norm_tol=1e-4, infeas_norm_tol=1e-1, max_iters=3000) if to_tol else \
            dict(gap_norm_tol=-1.0, infeas_norm_tol=-1.0, max_iters=int(rng.integers(10, 60)))
        X, y = O.gen_instance(kind, N, n, 0.1, int(rng.integers(1, 10**6)), pieces)
        P = R.prepare(X, y)
        r = R.papg(X, P.ys, feas_y=P.feas_y, feas_xi=P.feas_xi, threads=os.cpu_count() or 1, **kw)
        with crb.DualSolver(X, P.ys) as s:
            sg, _, _ = s.sigma_C()
            s.begin(crb.PapgConfig(sigma_C=r.sigma_C, **kw))
            stopped = False
            while not stopped:
                _, stopped = s.iterate(1 << 40)
            res, yg, xig, hist = s.finish()
            th = s.theta()
        same = (res.iters, res.restarts, res.reason) == (r.iters, r.restarts, O.REASONS_INV[r.reason])
        e = rel(th, r.theta), rel(yg, r.y)
        ok = same and e[0] <= 1e-12 and e[1] <= 1e-8 and abs(sg - r.sigma_C) <= 1e-10 * r.sigma_C
        bad += 0 if ok else 1
        worst = [max(worst[0], e[0]), max(worst[1], e[1])]
        print(f"{k:3d} {'ok ' if ok else 'BAD'} {kind:18s} N={N:4d} n={n:2d} iters={r.iters:4d} {r.reason:11s} "
              f"theta {e[0]:.1e} y {e[1]:.1e} sigma {abs(sg - r.sigma_C) / r.sigma_C:.1e}", flush=True)
    print(f"cases {cases}, failures {bad}, worst theta {worst[0]:.2e} y {worst[1]:.2e}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

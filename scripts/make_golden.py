"""Generates tests/golden/*.npz from the CPU oracle (oracle/cvxreg_oracle.c).

The reference has no golden vectors for this path; these
fixtures pin the oracle's own outputs (regression) and give the GPU tests
reference values that need no oracle run. Re-run only when the oracle's
algorithm intentionally changes:  python scripts/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

CASES = [
    # kind, N, n, noise, seed, pieces, iters, gap_tol, infeas_tol, B_theta, momentum
    ("sqnorm-uniform", 60, 5, 0.1, 1, 0, 40, -1.0, -1.0, 0.0, 1),
    ("maxaffine-uniform", 48, 10, 0.1, 2, 20, 30, -1.0, -1.0, 0.0, 1),
    ("lse-uniform", 40, 20, 0.05, 3, 50, 25, -1.0, -1.0, 0.0, 1),
    ("maxaffine-uniform", 33, 3, 0.1, 4, 5, 35, -1.0, -1.0, 3e-4, 1),   # ball binding
    ("sqnorm-uniform", 50, 2, 0.2, 5, 0, 30, -1.0, -1.0, 0.0, 0),       # DGA
    ("sqnorm-uniform", 80, 5, 0.1, 6, 0, 5000, 1e-6, 1e-1, 0.0, 1),     # to tolerance
]


def main():
    os.makedirs(OUT, exist_ok=True)
    d = {"count": np.array(len(CASES))}
    for i, (kind, N, n, noise, seed, pieces, iters, gt, it, B, mom) in enumerate(CASES):
        X, y = O.gen_instance(kind, N, n, noise, seed, pieces)
        p = O.prepare(X, y)
        s, _, _ = O.sigma_C(X)
        r = O.papg(X, p.ys, max_iters=iters, sigma_C=s, gap_norm_tol=gt, infeas_norm_tol=it,
                   B_theta=B, use_momentum=bool(mom), want_c_eta=True)
        d[f"X{i}"] = X
        d[f"ys{i}"] = p.ys
        d[f"meta{i}"] = np.array([iters, s, gt, it, B, mom], np.float64)
        d[f"theta{i}"] = r.theta
        d[f"c_eta{i}"] = r.c_eta
        d[f"y{i}"] = r.y
        d[f"xi{i}"] = r.xi
        d[f"hist{i}"] = r.history[:, :7]
        d[f"iters{i}"] = np.array([r.iters, r.restarts])
        d[f"scal{i}"] = np.array([r.g_final, r.delta_estimate, r.B_theta])
        print(kind, N, n, "iters", r.iters, r.reason, "restarts", r.restarts)
    np.savez_compressed(os.path.join(OUT, "papg_small.npz"), **d)
    np.savez_compressed(
        os.path.join(OUT, "rng.npz"),
        raw_1_2=O.rng_draws(1, 2, 8, "raw53"),
        normal_5eed_97=O.rng_draws(0x5EED, 97, 8, "normal"),
        uniform_7_3=O.rng_draws(7, 3, 8, "uniform"),
    )


if __name__ == "__main__":
    main()

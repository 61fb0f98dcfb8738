"""Runs the REFERENCE's own compiled papg_solve (oracle/_ref, singleton blocks) on the
BASELINE configurations it can hold in host memory and stores what a GPU test needs to
compare against: y, xi, the history, iteration count / reason, sigma_C and sampled rows
of theta (the full theta is 0.8 GB at config 2, 3.2 GB at config 3).

    python scripts/make_ref_baseline_golden.py cfg1|cfg2|cfg3

The reference estimates sigma_C itself with single-threaded O(N^2 n) passes: config 1
takes about a minute, config 2 about 15 minutes, config 3 (10 iterations) about 40.
Output: tests/golden/ref_baseline_<cfg>.npz.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402  (BASELINE generator kinds: inputs only)
from oracle import ref as R  # noqa: E402

RUNS = {  # max_iters, gap_norm_tol, infeas_norm_tol
    "cfg1": (2000, -1.0, -1.0),     # BASELINE: 2000 iterations
    "cfg2": (100000, 1e-4, 1e-1),   # BASELINE: to dual-gap tolerance 1e-4
    "cfg3": (10, -1.0, -1.0),       # fixed k
}
SAMPLE_ROWS = 12


def main():
    name = sys.argv[1]
    cfg = bench.CONFIGS[name]
    iters, gt, ft = RUNS[name]
    N, n = cfg["N"], cfg["n"]
    X, y = O.gen_instance(cfg["kind"], N, n, cfg["noise"], 1, cfg["pieces"])
    P = R.prepare(X, y)
    t0 = time.time()
    r = R.papg(X, P.ys, feas_y=P.feas_y, feas_xi=P.feas_xi, max_iters=iters, gap_norm_tol=gt,
               infeas_norm_tol=ft, threads=os.cpu_count() or 1)
    spent = time.time() - t0
    rows = np.unique(np.linspace(0, N - 1, SAMPLE_ROWS).astype(np.int64))
    cross = r.theta[: N * (N - 1)].reshape(N, N - 1)
    out = dict(
        ys=P.ys, rows=rows, theta_rows=cross[rows].copy(), theta_pos=r.theta[N * (N - 1):].copy(),
        theta_norm=np.array(np.linalg.norm(r.theta)), y=r.y, xi=r.xi, hist=r.history[:, :7],
        iters=np.array([r.iters, r.restarts, O.REASONS_INV[r.reason], int(r.saturated)]),
        scal=np.array([r.g_final, r.delta_estimate, r.B_theta, r.L_g, r.sigma_C]),
        meta=np.array([iters, gt, ft]), seconds=np.array(spent),
        loop_seconds=np.array(r.history[-1, 7] - r.history[0, 7]),
    )
    path = os.path.join(ROOT, "tests", "golden", f"ref_baseline_{name}.npz")
    np.savez_compressed(path, **out)
    print(name, "iters", r.iters, r.reason, "sigma_C", r.sigma_C, f"{spent:.0f} s",
          "per iteration", (r.history[-1, 7] - r.history[0, 7]) / max(r.iters - 1, 1), flush=True)


if __name__ == "__main__":
    main()

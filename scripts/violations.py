"""Fraction of violated rows (C eta < 0) and of 8x32 warp-stages with a violation or a live multiplier."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1407_7220_b200 as crb

d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", 10, 10000, 0.1, 1, 20))
prep = crb.prepare_problem(d)
N = 10000
with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
    sig = s.sigma_C()[0]
    s.begin(crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig))
    done = 0
    for target in [50, 200, 1000, 1500]:
        s.iterate(target - done)
        done = target
        rows = s.rows()[: N * (N - 1)]
        th = s.theta()[: N * (N - 1)]
        mask = ~np.eye(N, dtype=bool)
        V = np.zeros((N, N)); V[mask] = rows
        T = np.zeros((N, N)); T[mask] = th
        hot = (V < 0) | (T != 0)
        st = hot[: N // 8 * 8, : N // 32 * 32].reshape(N // 8, 8, N // 32, 32).any(axis=(1, 3))
        print(f"iter {target}: violated {np.mean(V[mask] < 0):.4f} live {np.mean(th != 0):.4f} hot 8x32 stages {st.mean():.3f}", flush=True)

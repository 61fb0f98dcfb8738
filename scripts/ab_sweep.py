"""A/B of sweep library variants at cfg 2: mean per-launch sweep time (CUDA
events, every launch) over iterations 6..K, best of R runs.
    CRB_LIB=ab/x.so python scripts/ab_sweep.py [K] [R] [N] [n]"""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_1407_7220_b200 as crb

K = int(sys.argv[1]) if len(sys.argv) > 1 else 25
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
n = int(sys.argv[4]) if len(sys.argv) > 4 else 10
d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", n, N, 0.1, 1, 20))
prep = crb.prepare_problem(d)
with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
    sig = s.sigma_C()[0]
    cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig)
    best = None
    for _ in range(R):
        s.begin(cfg)
        s.iterate(K)
        t = s.last_sweep_times() * 1e6
        step = s.last_timing()[0] / K * 1e6
        if best is None or t[5:].mean() < best[0]:
            best = (t[5:].mean(), t[:5].mean(), step, t)
    res = s.finish() if hasattr(s, "finish") else None
print(f"{os.path.basename(os.environ.get('CRB_LIB', 'default'))}: sweeps 6..{K} {best[0]:.1f} us "
      f"(1..5 {best[1]:.1f}), step {best[2]:.1f} us; per launch "
      + " ".join(f"{x:.0f}" for x in best[3]))

"""Fraction of zero multipliers and of all-zero tiles in the dual store over iterations."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1407_7220_b200 as crb

cfgs = {"cfg2": ("maxaffine-uniform", 10000, 10, 20, 0.1), "cfg1": ("sqnorm-uniform", 1000, 5, 0, 0.1),
        "cfg3": ("lse-uniform", 20000, 20, 50, 0.05)}
kind, N, n, pieces, noise = cfgs[sys.argv[1]]
d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, noise, 1, pieces))
prep = crb.prepare_problem(d)
with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
    sig = s.sigma_C()[0]
    s.begin(crb.PapgConfig(max_iters=100000, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig))
    done = 0
    for target in [1, 5, 20, 100, 500, 2000]:
        s.iterate(target - done)
        done = target
        th = s.theta()[: N * (N - 1)]
        full = np.zeros((N, N))
        mask = ~np.eye(N, dtype=bool)
        full[mask] = th
        nz = full != 0
        out = [f"iter {target}: nonzero {nz.mean():.4f}"]
        for (tr, tc) in [(8, 32), (8, 224), (32, 32)]:
            R = N // tr * tr
            C = N // tc * tc
            t = nz[:R, :C].reshape(R // tr, tr, C // tc, tc).any(axis=(1, 3))
            out.append(f"tiles {tr}x{tc} nonzero {t.mean():.4f}")
        print("  ".join(out), flush=True)

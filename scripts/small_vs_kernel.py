"""Persistent small-N loop vs the per-kernel path (graphs) at small N: us/iteration."""
import os, sys
sys.path.insert(0, ".")
import paper_1407_7220_b200 as crb
for N, n in [(300, 5), (600, 5), (1000, 5), (1500, 5), (2000, 5), (1000, 10)]:
    d = crb.gen_instance(crb.GeneratorSpec("sqnorm-uniform", n, N, 0.1, 1))
    p = crb.prepare_problem(d)
    out = []
    for small in ("1", "0"):
        os.environ["CRB_SMALL"] = small
        with crb.DualSolver(p.data.xs, p.data.ys) as s:
            cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=75.0)
            s.begin(cfg)
            s.iterate(50)
            s.begin(cfg)
            s.iterate(1000)
            out.append(s.last_timing()[0] / 1000 * 1e6)
    print(f"N={N} n={n}: small {out[0]:.2f} us, per-kernel {out[1]:.2f} us")

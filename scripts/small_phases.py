"""cfg 1 on the persistent small-N loop: per-iteration time over 2000 iterations
and the phase breakdown of the first iterations (CRB_SMALL_TRACE=1)."""
import os, sys
sys.path.insert(0, ".")
import paper_1407_7220_b200 as crb
d = crb.gen_instance(crb.GeneratorSpec("sqnorm-uniform", 5, 1000, 0.1, 1))
p = crb.prepare_problem(d)
with crb.DualSolver(p.data.xs, p.data.ys) as s:
    cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=75.04526292327877)
    s.begin(cfg)
    s.iterate(60)
    s.begin(cfg)
    s.iterate(2000)
    sec = s.last_timing()[0]
    print(f"cfg1 small loop: {sec / 2000 * 1e6:.2f} us/iteration over 2000 iterations")

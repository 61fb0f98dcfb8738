"""ncu target: cfg 1 on the persistent small-N loop, launches of 64 iterations."""
import sys
sys.path.insert(0, ".")
import paper_1407_7220_b200 as crb
d = crb.gen_instance(crb.GeneratorSpec("sqnorm-uniform", 5, 1000, 0.1, 1))
p = crb.prepare_problem(d)
with crb.DualSolver(p.data.xs, p.data.ys) as s:
    cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=75.04526292327877)
    s.begin(cfg)
    for _ in range(4):
        s.iterate(64)
    print("done", s.iterate(0)[0])

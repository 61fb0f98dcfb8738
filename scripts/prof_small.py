"""c1 run in persistent small-N mode for ncu (dev tool)."""
import sys
sys.path.insert(0, '.')
import paper_1407_7220_b200 as crb
d = crb.gen_instance(crb.GeneratorSpec("sqnorm-uniform", 5, 1000, 0.1, 1))
p = crb.prepare_problem(d)
s = crb.DualSolver(p.data.xs, p.data.ys)
s.begin(crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=75.0))
s.iterate(50)
print("ok", s.last_timing())

"""Short run of one config for ncu: a few iterations in direct-launch mode."""
import sys
sys.path.insert(0, '.')
import paper_1407_7220_b200 as crb
kind, N, n, pieces, noise = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 4
d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, noise, 1, pieces))
prep = crb.prepare_problem(d)
s = crb.DualSolver(prep.data.xs, prep.data.ys)
cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=300.0, graph_iters=-1)
s.begin(cfg)
s.iterate(iters)
print("ok", s.last_timing())

"""Time to tolerance through papg_solve, repeated (median), cfg 2 (dev tool)."""
import sys, time, statistics
sys.path.insert(0, '.')
import paper_1407_7220_b200 as crb
d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", 10, 10000, 0.1, 1, 20))
p = crb.prepare_problem(d)
ts, sg = [], []
for rep in range(7):
    cfg = crb.PapgConfig(gap_norm_tol=1e-4, infeas_norm_tol=1e-1, record_history=False)
    t0 = time.perf_counter()
    r = crb.papg_solve(p, cfg, want_dual=False)
    ts.append(time.perf_counter() - t0)
    sg.append(r.sigma_seconds)
print(f"ttt median {1e3*statistics.median(ts[1:]):.2f} ms (min {1e3*min(ts[1:]):.2f}), sigma median {1e3*statistics.median(sg[1:]):.2f} ms, iters {r.report.iters}")

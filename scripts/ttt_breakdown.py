"""Breakdown of a cfg2 time-to-tolerance solve through the public API (dev tool)."""
import sys, time
sys.path.insert(0, '.')
import paper_1407_7220_b200 as crb
d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", 10, 10000, 0.1, 1, 20))
p = crb.prepare_problem(d)
for rep in range(3):
    t0 = time.perf_counter()
    s = crb.DualSolver(p.data.xs, p.data.ys)
    t1 = time.perf_counter()
    cfg = crb.PapgConfig(gap_norm_tol=1e-4)
    s.begin(cfg)
    t2 = time.perf_counter()
    done, stopped = s.iterate(1 << 30)
    t3 = time.perf_counter()
    res, y, xi, hist = s.finish()
    t4 = time.perf_counter()
    s.close()
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms, begin(+sigma {1e3*res.sigma_seconds:.1f}) {1e3*(t2-t1):.1f} ms, "
          f"iterate {done} its {1e3*(t3-t2):.1f} ms, finish {1e3*(t4-t3):.1f} ms, close {1e3*(t5-t4):.1f} ms, total {1e3*(t5-t0):.1f}")

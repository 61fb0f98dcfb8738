import os, sys, time
sys.path.insert(0, ".")
import paper_1407_7220_b200 as crb
for N, n in [(10000, 10), (20000, 20), (100000, 5)]:
    d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", n, N, 0.1, 1, 10))
    prep = crb.prepare_problem(d)
    with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
        s.sigma_C()
        t = time.perf_counter(); r = s.sigma_C(); dt = time.perf_counter() - t
        print(f"grid={os.environ.get('CRB_POWER_GRID','148')} N={N} n={n} sigma={r[0]:.12g} steps={r[1]} {dt*1e3:.2f} ms", flush=True)

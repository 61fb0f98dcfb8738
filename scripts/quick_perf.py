import sys, time; sys.path.insert(0, '.')
import numpy as np
import paper_1407_7220_b200 as crb
for (kind, N, n, pieces, noise) in [("sqnorm-uniform", 1000, 5, 0, 0.1), ("maxaffine-uniform", 10000, 10, 20, 0.1)]:
    d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, noise, 1, pieces))
    prep = crb.prepare_problem(d)
    s = crb.DualSolver(prep.data.xs, prep.data.ys)
    t = time.time(); sig = s.sigma_C(); print(kind, N, "sigma", sig, time.time()-t, flush=True)
    cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig[0])
    s.begin(cfg)
    s.iterate(10)
    for k in [50, 200]:
        s.iterate(k)
        sec, launches, sw = s.last_timing()
        print(f"  {k} iters: {sec*1e3:.2f} ms total, {sec/k*1e6:.1f} us/iter, sweep {sw/k*1e6 if sw else 0:.1f} us, {N*N*k/sec/1e9:.1f} Gpair/s, launches {launches}", flush=True)
    print("  time_sweep", s.time_sweep(20)*1e6, "us", flush=True)
    s.close()

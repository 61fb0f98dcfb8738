"""ALCC (f1) throughput: device time per MAPG iteration and the penalty sweep alone."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np
import paper_1407_7220_b200 as crb

CFG = {"cfg1": ("sqnorm-uniform", 1000, 5, 0.1, 0), "cfg2": ("maxaffine-uniform", 10000, 10, 0.1, 20),
       "cfg3": ("lse-uniform", 20000, 20, 0.05, 50), "n5": ("maxaffine-uniform", 10000, 5, 0.1, 20)}
for name in sys.argv[1:]:
    kind, N, n, noise, pieces = CFG[name]
    data = crb.gen_instance(crb.GeneratorSpec(kind, n, N, noise, 1, pieces))
    prep = crb.prepare_problem(data)
    with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
        t0 = time.perf_counter()
        s1 = s.sigma_A(1); s2 = s.sigma_A(2)
        ts = time.perf_counter() - t0
        cfg = crb.AlccConfig(max_outer=3, mapg_cap=300, infeas_norm_tol=-1.0, alpha1_scale=1e-30, sigma_A1=s1[0], sigma_A2=s2[0])
        res, y, xi, hist, mi = s.alcc(cfg, prep.bounds, prep.feasible)
        t0 = time.perf_counter()
        res, y, xi, hist, mi = s.alcc(cfg, prep.bounds, prep.feasible)
        wall = time.perf_counter() - t0
        sw = s.time_penalty_sweep(20)
    it = res.mapg_iters_total
    per = res.mapg_seconds / it
    print(json.dumps(dict(cfg=name, N=N, n=n, sigma_s=ts, sigma_iters=[s1[1], s2[1]], mapg=list(map(int, mi)),
                          mapg_us=per * 1e6, sweep_us=sw * 1e6, sweep_gbs=8 * N * N / sw / 1e9,
                          sweep_share=sw / per, pair_evals_per_s=N * N / per, wall=wall,
                          launches=int(res.launches))), flush=True)

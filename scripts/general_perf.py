"""General-K P-APG(ALCC) timing: dual iterations with bounded inner ALCC (dev tool)."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np
import paper_1407_7220_b200 as crb

N, n, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 2
d = crb.gen_instance(crb.GeneratorSpec("sqnorm-uniform", n, N, 0.1, 1, 0))
prep = crb.prepare_problem(d)
inner = crb.AlccConfig(max_outer=3, mapg_cap=300)
with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
    t0 = time.perf_counter()
    s.set_partition(K, prep.feasible, inner)
    t_part = time.perf_counter() - t0
    t0 = time.perf_counter()
    sig = s.sigma_C()
    t_sig = time.perf_counter() - t0
    cfg = crb.PapgConfig(K=K, inner=inner, max_iters=iters, gap_norm_tol=-1.0, sigma_C=sig[0])
    s.begin(cfg)
    t0 = time.perf_counter()
    s.iterate(1 << 30)
    t_it = time.perf_counter() - t0
    st = s.partition_stats()
    sec, launches, sw = s.last_timing()
print(json.dumps(dict(N=N, n=n, K=K, nbar=N // K, partition_s=t_part, sigma_s=t_sig, sigma_steps=sig[1],
                      iter_s=t_it / iters, inner_mapg=st["inner_iters"], inner_s=st["inner_seconds"],
                      us_per_mapg=st["inner_seconds"] / max(st["inner_iters"], 1) * 1e6,
                      cross_sweep_ms=sw / iters * 1e3)))

"""Quick per-iteration timing of the dual loop for a few configs (dev tool)."""
import sys, time
sys.path.insert(0, '.')
import paper_1407_7220_b200 as crb
CONFIGS = {
    "c1": ("sqnorm-uniform", 1000, 5, 0, 0.1),
    "c2": ("maxaffine-uniform", 10000, 10, 20, 0.1),
    "c2n5": ("sqnorm-uniform", 10000, 5, 0, 0.1),
    "c3": ("lse-uniform", 20000, 20, 50, 0.05),
}
names = sys.argv[1:] or ["c1", "c2"]
for name in names:
    kind, N, n, pieces, noise = CONFIGS[name]
    d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, noise, 1, pieces))
    prep = crb.prepare_problem(d)
    s = crb.DualSolver(prep.data.xs, prep.data.ys)
    t = time.time(); sig = s.sigma_C(); ts = time.time() - t
    print(f"{name} N={N} n={n} sigma={sig[0]:.6f} ({sig[1]} steps, {ts*1e3:.1f} ms)", flush=True)
    for gi in ([0, -1] if N <= 2000 else [-1]):
        cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig[0], graph_iters=gi)
        s.begin(cfg)
        s.iterate(10)
        k = 200
        s.iterate(k)
        sec, launches, sw = s.last_timing()
        print(f"  mode={'graph' if gi >= 0 else 'direct'} {k} iters: {sec/k*1e6:.1f} us/iter"
              f" sweep {sw/k*1e6:.1f} us  {N*N*k/sec/1e9:.1f} Gpair/s (sweep-only {N*N/(sw/k)/1e9 if sw else 0:.1f})"
              f" HBM {24*N*N/(sw/k)/1e12 if sw else 0:.2f} TB/s launches {launches}", flush=True)
    s.close()

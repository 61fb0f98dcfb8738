"""Sweep time per n at early / mid / late iterations (N from argv, maxaffine data).

    python scripts/phase_perf.py N n1 n2 ...
"""
import os, sys
sys.path.insert(0, ".")
import paper_1407_7220_b200 as crb
N = int(sys.argv[1])
for n in [int(a) for a in sys.argv[2:]]:
    d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", n, N, 0.1, 1, 20))
    prep = crb.prepare_problem(d)
    with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
        sig = s.sigma_C()[0]
        s.begin(crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig, graph_iters=-1))
        out = []
        done = 0
        for lo, hi in [(0, 10), (10, 50), (50, 300), (300, 500), (500, 1000), (1000, 2000)]:
            s.iterate(hi - lo)
            sec, launches, sw = s.last_timing()
            out.append(f"[{lo},{hi}) {sw/(hi-lo)*1e6:.1f}")
        print(f"{os.environ.get('TAG','')} N={N} n={n} {s.sweep_variant} sweep us: " + "  ".join(out), flush=True)

"""Sweep time per n (N = 10000, late iterations) for the selected kernel variant."""
import os, sys
sys.path.insert(0, ".")
import paper_1407_7220_b200 as crb
for n in [int(a) for a in sys.argv[1:]]:
    d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", n, 10000, 0.1, 1, 20))
    prep = crb.prepare_problem(d)
    with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
        sig = s.sigma_C()[0]
        s.begin(crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig, graph_iters=-1))
        s.iterate(300)
        s.iterate(200)
        sec, launches, sw = s.last_timing()
        print(f"{os.environ.get('TAG','')} n={n} variant={s.sweep_variant} sweep {sw/200*1e6:.1f} us iter {sec/200*1e6:.1f} us", flush=True)

"""cfg 2 step time, iterations 6..25: direct launches (per-sweep events / none) vs CUDA graphs."""
import os, sys
sys.path.insert(0, ".")
import paper_1407_7220_b200 as crb
d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", 10, 10000, 0.1, 1, 20))
p = crb.prepare_problem(d)
with crb.DualSolver(p.data.xs, p.data.ys) as s:
    sig = s.sigma_C()[0]
    for gi, ev in [(-1, None), (-1, "0"), (4, None), (20, None), (4, "G"), (20, "G")]:
        if ev == "G":
            os.environ["CRB_GRAPH_EVENTS"] = "1"
        if ev == "G":
            pass
        elif ev is None:
            os.environ.pop("CRB_SWEEP_EVENTS", None)
        else:
            os.environ["CRB_SWEEP_EVENTS"] = ev
        best = 1e9
        for _ in range(3):
            s.begin(crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig,
                                   graph_iters=gi))
            s.iterate(5)
            s.iterate(20)
            best = min(best, s.last_timing()[0] / 20 * 1e6)
        print(f"graph_iters={gi} events={ev}: {best:.1f} us/step (iterations 6..25)")

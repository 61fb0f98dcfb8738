"""cfg 1 on the persistent small-N loop: per-iteration time over 2000 iterations
and the phase breakdown (CRB_TRACE=1 prints the mean phase durations of the
first 63 iterations of every launch: early, around 500, around 1500)."""
import os, sys
sys.path.insert(0, ".")
os.environ["CRB_TRACE"] = "1"
import paper_1407_7220_b200 as crb
d = crb.gen_instance(crb.GeneratorSpec("sqnorm-uniform", 5, 1000, 0.1, 1))
p = crb.prepare_problem(d)
with crb.DualSolver(p.data.xs, p.data.ys) as s:
    cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=75.04526292327877)
    s.begin(cfg)
    for k in (64, 436, 64, 936, 64):
        s.iterate(k)
        print(f"  ^ launch of {k} iterations ending at {s.iterate(0)[0]}: {s.last_timing()[0] / k * 1e6:.2f} us/iteration" if False else f"  ^ {k} iterations", flush=True)
    os.environ.pop("CRB_TRACE")
    s.begin(cfg)
    s.iterate(60)
    s.begin(cfg)
    s.iterate(2000)
    sec = s.last_timing()[0]
    print(f"cfg1 small loop: {sec / 2000 * 1e6:.2f} us/iteration over 2000 iterations")

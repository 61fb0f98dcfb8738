"""Tiny solves for compute-sanitizer runs (memcheck / racecheck / synccheck):
the DMMA/TMA pair sweep ring (CRB_SMALL=0), the persistent small-N loop, the
sigma power loops (cluster and grid), the fused reduce+primal (CRB_FUSE=1),
the ALCC penalty sweeps and a general-K partition.
    python scripts/sanitize_cases.py <case>"""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import paper_1407_7220_b200 as crb

case = sys.argv[1] if len(sys.argv) > 1 else "sweep"


def inst(N, n, kind="maxaffine-uniform", pieces=5):
    d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, 0.1, 3, pieces))
    return crb.prepare_problem(d)


if case in ("sweep", "small", "fused"):
    if case != "small":
        os.environ["CRB_SMALL"] = "0"
    if case == "fused":
        os.environ["CRB_FUSE"] = "1"
    p = inst(700, 10) if case != "small" else inst(300, 5)
    r = crb.papg_solve(p, crb.PapgConfig(max_iters=6, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                                         sigma_C=50.0))
    print(case, "iters", r.report.iters, "y0", r.point.y[0])
elif case in ("sigma", "sigma_grid"):
    if case == "sigma_grid":
        os.environ["CRB_SIGMA_CLUSTER"] = "0"
    p = inst(900, 8)
    with crb.DualSolver(p.data.xs, p.data.ys) as s:
        print(case, s.sigma_C(max_iters=30))
elif case == "alcc":
    p = inst(400, 5)
    r = crb.alcc_solve(p, crb.AlccConfig(max_outer=2, mapg_cap=5))
    print(case, "outer", r.outer_iters)
elif case == "general":
    p = inst(200, 3)
    r = crb.papg_solve(p, crb.PapgConfig(K=2, max_iters=2, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                                         sigma_C=50.0, inner=crb.AlccConfig(max_outer=1, mapg_cap=5)))
    print(case, "iters", r.report.iters)

import os, sys
sys.path.insert(0, ".")
import numpy as np
from oracle import oracle as O
import paper_1407_7220_b200 as crb
os.environ["CRB_SIGMA"] = "sweep"
for var in ("dfma", "mma"):
    os.environ["CRB_SWEEP"] = var
    for kind, N, n, pieces in [("sqnorm-uniform", 400, 5, 0), ("maxaffine-uniform", 300, 10, 20),
                               ("lse-uniform", 250, 20, 50), ("quadratic", 333, 1, 0),
                               ("exponential", 150, 24, 0)]:
        X, y = O.gen_instance(kind, N, n, 0.1, 3, pieces)
        p = O.prepare(X, y)
        so, ito, co = O.sigma_C(X)
        with crb.DualSolver(X, p.ys) as d:
            sg, itg, cg = d.sigma_C()
        print(var, kind, n, so, sg, ito, itg, (sg - so) / so, flush=True)

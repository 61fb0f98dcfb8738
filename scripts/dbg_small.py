import sys, os; sys.path.insert(0, '.')
import numpy as np
import paper_1407_7220_b200 as crb
from oracle import oracle as O
for n in [5, 12, 13, 16, 20, 24]:
    for N in [40, 64, 127]:
        if N < n + 1: continue
        X, y = O.gen_instance("maxaffine-uniform", N, n, 0.1, 3, 5)
        p = O.prepare(X, y)
        cfg = crb.PapgConfig(max_iters=20, sigma_C=float(O.sigma_C(X)[0]), gap_norm_tol=-1, infeas_norm_tol=-1)
        try:
            with crb.DualSolver(X, p.ys) as d:
                d.begin(cfg)
                done, st = d.iterate(1 << 30)
                print(n, N, "ok", done)
        except Exception as e:
            print(n, N, "ERR", e)

import sys, os; sys.path.insert(0, '.')
import numpy as np
import paper_1407_7220_b200 as crb
g = np.load('tests/golden/papg_small.npz')
for i in range(int(g["count"])):
    X, ys = g[f"X{i}"], g[f"ys{i}"]
    it, s, gt, ft, B, mom = g[f"meta{i}"]
    cfg = crb.PapgConfig(max_iters=int(it), sigma_C=float(s), gap_norm_tol=float(gt), infeas_norm_tol=float(ft), B_theta=float(B))
    try:
        with crb.DualSolver(X, ys) as d:
            d.begin(cfg, bool(mom))
            done, st = d.iterate(1 << 30)
            th = d.theta()
            print(i, X.shape, os.environ.get("CRB_SMALL"), "ok", done, np.linalg.norm(th - g[f"theta{i}"]) / np.linalg.norm(g[f"theta{i}"]))
    except Exception as e:
        print(i, X.shape, os.environ.get("CRB_SMALL"), "ERR", e)

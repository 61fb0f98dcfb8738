"""Debug: ALCC GPU vs oracle divergence per outer step count."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import oracle as O
import paper_1407_7220_b200 as crb

kind, N, n, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
X, y = O.gen_instance(kind, N, n, 0.2, seed, 0 if kind == "sqnorm-uniform" else 3)
P = O.prepare(X, y, 1e-3)
s1, s2 = O.sigma_A(X, 1)[0], O.sigma_A(X, 2)[0]
bounds = crb.ProblemBounds(P.B_theta, P.Bbar_y, P.Bbar_xi, P.gamma)
for mo in range(1, 6):
    for cap in (50, 400, 4000):
        o = O.alcc(X, P.ys, gamma=P.gamma, Bbar_y=P.Bbar_y, Bbar_xi=P.Bbar_xi, warm_y=P.feas_y,
                   warm_xi=P.feas_xi, sigma_A1=s1, sigma_A2=s2, max_outer=mo, mapg_cap=cap)
        with crb.DualSolver(X, P.ys, P.gamma) as s:
            res, gy, gxi, hist, mi = s.alcc(crb.AlccConfig(sigma_A1=s1, sigma_A2=s2, max_outer=mo,
                                                           mapg_cap=cap), bounds,
                                            crb.PrimalPoint(P.feas_y, P.feas_xi))
        e = np.linalg.norm(gy - o.y) / np.linalg.norm(o.y)
        print(mo, cap, list(mi), list(o.mapg_iters), f"{e:.3e}", o.reason, flush=True)

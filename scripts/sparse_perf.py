"""Per-iteration sweep time over the solve (masked vs dense dual store), cfg 2."""
import os, sys
sys.path.insert(0, ".")
import paper_1407_7220_b200 as crb

kind, N, n, pieces = ("maxaffine-uniform", 10000, 10, 20) if len(sys.argv) < 2 else (sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
d = crb.gen_instance(crb.GeneratorSpec(kind, n, N, 0.1, 1, pieces))
prep = crb.prepare_problem(d)
with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
    sig = s.sigma_C()[0]
    s.begin(crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig, graph_iters=-1))
    done = 0
    for a, b in [(0, 10), (10, 50), (50, 200), (200, 1000), (1000, 2000)]:
        s.iterate(b - done)
        done = b
        sec, launches, sw = s.last_timing()
        k = b - a
        print(f"{os.environ.get('CRB_SPARSE', '1')} iters {a}-{b}: {sec / k * 1e6:.1f} us/iter, sweep {sw / k * 1e6:.1f} us", flush=True)

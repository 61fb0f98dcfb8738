"""Randomised check of the GPU-count-invariant mode: for random (N, n, D) the iterates of p
shard handles (host-emulated allgather) are bitwise those of one handle, for every p | D.

    python scripts/fuzz_canonical.py [cases] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1407_7220_b200 as crb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_gpu_canonical import run_shards  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 25
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
    bad = 0
    for k in range(cases):
        n = int(rng.choice([1, 3, 5, 10, 16, 20, 32]))
        D = int(rng.choice([2, 4, 6, 8, 12, 16]))
        N = int(rng.integers(max(n + 1, 8 * D), 700))
        iters = int(rng.integers(3, 25))
        kind, pieces = [("sqnorm-uniform", 0), ("maxaffine-uniform", 9), ("lse-uniform", 15)][rng.integers(3)]
        X, y = O.gen_instance(kind, N, n, 0.1, int(rng.integers(1, 10**6)), pieces)
        ys = O.prepare(X, y).ys
        cfg = crb.PapgConfig(max_iters=iters, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                             sigma_C=float(rng.uniform(20, 200)))
        ps = [p for p in range(1, D + 1) if D % p == 0]
        base = run_shards(X, ys, cfg, 1, D, iters)
        ok = np.linalg.norm(base["theta"]) > 0
        for p in ps[1:]:
            r = run_shards(X, ys, cfg, p, D, iters)
            ok = ok and all(np.array_equal(r[key], base[key]) for key in ("theta", "y", "xi", "hist"))
        bad += 0 if ok else 1
        print(f"{k:3d} {'ok ' if ok else 'BAD'} {kind:18s} N={N:4d} n={n:2d} D={D:2d} p={ps} iters={iters}",
              flush=True)
    print(f"cases {cases}, failures {bad}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

"""Strong-scaling projection on ONE GPU (the build has no second GPU): the p row shards of
a BASELINE config run as p handles on the same device with the per-iteration exchange done
on the host (exact iterates, as in the sharded emulation tests), and every shard's local
phase (primal + sweep + reduce over its N/p rows) is timed on its own. With one GPU per
shard the step time is max over shards of the local phase + the allreduce of the payload,
so  speed-up(p) ~ t_local(1) / (max_r t_local(r, p) + t_exchange(p)).  The exchange term is
modelled from the payload size (NCCL ring allreduce over NVLink 5, 2 (p-1)/p x bytes at
the stated bus bandwidth + a launch latency); it is NOT measured.

    python scripts/shard_scaling_probe.py cfg3|cfg4|cfg2 [iters]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1407_7220_b200 as crb  # noqa: E402

NVLINK_BUS_GBS = 350.0   # conservative NCCL allreduce bus bandwidth for ~MB messages on NVLink 5
LAUNCH_US = 25.0         # NCCL kernel launch + sync latency


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    warm = 5
    cfg = bench.CONFIGS[name]
    N, n = cfg["N"], cfg["n"]
    data = crb.gen_instance(crb.GeneratorSpec(cfg["kind"], n, N, cfg["noise"], 1, cfg["pieces"]))
    prep = crb.prepare_problem(data)
    pc = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                        sigma_C=bench.SIGMA_C[name], graph_iters=-1)
    base = None
    for p in (1, 2, 4, 8):
        shards = [crb.DualSolver(prep.data.xs, prep.data.ys, row_begin=N * r // p,
                                 row_end=N * (r + 1) // p) for r in range(p)]
        try:
            for d in shards:
                d.begin(pc)
            local = np.zeros((iters, p))
            for it in range(warm + iters):
                for r, d in enumerate(shards):
                    t0 = time.perf_counter()
                    d.iter_local()  # enqueue + stream synchronize
                    if it >= warm:
                        local[it - warm, r] = time.perf_counter() - t0
                total = sum(d.exchange_get() for d in shards)
                for d in shards:
                    d.exchange_put(total)
                for d in shards:
                    d.iter_finish()
            t_local = np.median(local, axis=0).max()
            payload = 8.0 * (N * (n + 2) + 5)
            t_x = 0.0 if p == 1 else (2.0 * (p - 1) / p * payload / (NVLINK_BUS_GBS * 1e9) + LAUNCH_US * 1e-6)
            if base is None:
                base = t_local
            print(f"{name} p={p}: rows/shard {N // p}, local phase {t_local * 1e3:.3f} ms (max over shards, "
                  f"median of {iters} iterations {warm + 1}..{warm + iters}), modelled exchange "
                  f"{t_x * 1e6:.0f} us ({payload / 1e6:.2f} MB payload) -> projected step "
                  f"{(t_local + t_x) * 1e3:.3f} ms, speed-up {base / (t_local + t_x):.2f}x, "
                  f"efficiency {base / (t_local + t_x) / p:.2f}", flush=True)
        finally:
            for d in shards:
                d.close()


if __name__ == "__main__":
    main()

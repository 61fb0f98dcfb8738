"""Cost of the GPU-count-invariant mode (cr_set_canonical_blocks) on one GPU:
ms per dual iteration of a BASELINE config, default path vs D canonical blocks.
    python scripts/canon_perf.py [cfg2] [D ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1407_7220_b200 as crb  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    Ds = [int(a) for a in sys.argv[2:]] or [0, 1, 2, 4, 8]
    cfg = bench.CONFIGS[name]
    data = crb.gen_instance(crb.GeneratorSpec(cfg["kind"], cfg["n"], cfg["N"], cfg["noise"], 1,
                                              cfg["pieces"]))
    prep = crb.prepare_problem(data)
    pc = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                        sigma_C=bench.SIGMA_C[name])
    with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
        for D in Ds:
            s.set_canonical_blocks(D)
            s.begin(pc)
            s.iterate(5)
            best = 1e9
            for _ in range(3):
                s.begin(pc)
                s.iterate(5)
                s.iterate(20)
                sec, k, sw = s.last_timing()
                best = min(best, sec / 20)
            print(f"{name} D={D}: {best * 1e3:.4f} ms/iteration (iterations 6-25), "
                  f"{cfg['N'] ** 2 / best / 1e9:.1f} G pair-updates/s", flush=True)


if __name__ == "__main__":
    main()

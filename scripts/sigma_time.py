"""sigma_C wall time per config (cluster vs grid path): python scripts/sigma_time.py cfg..."""
import os, sys, time
sys.path.insert(0, ".")
import bench
import paper_1407_7220_b200 as crb
for name in sys.argv[1:] or ["cfg1", "cfg2"]:
    c = bench.CONFIGS[name]
    d = crb.gen_instance(crb.GeneratorSpec(c["kind"], c["n"], c["N"], c["noise"], 1, c["pieces"]))
    prep = crb.prepare_problem(d)
    with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
        out = []
        for _ in range(4):
            t0 = time.perf_counter()
            sg, it, cv = s.sigma_C()
            out.append(time.perf_counter() - t0)
    print(f"{name} {os.environ.get('CRB_SIGMA_CLUSTER', 'default')}: sigma {sg!r} steps {it} "
          f"conv {cv} seconds {min(out) * 1e3:.3f} ms (of {[round(x * 1e3, 3) for x in out]})")

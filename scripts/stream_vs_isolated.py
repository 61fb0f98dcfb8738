"""cfg 2 sweep: per-launch CUDA-event durations in one stream of iterations vs
the same iterations issued one call (host sync) at a time, plus SM clock
samples, to separate steady-state effects (power, write-back overlap) from the
kernel itself.   python scripts/stream_vs_isolated.py [iters]"""
import subprocess, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1407_7220_b200 as crb

K = int(sys.argv[1]) if len(sys.argv) > 1 else 25
d = crb.gen_instance(crb.GeneratorSpec("maxaffine-uniform", 10, 10000, 0.1, 1, 20))
prep = crb.prepare_problem(d)
with crb.DualSolver(prep.data.xs, prep.data.ys) as s:
    sig = s.sigma_C()[0]
    cfg = crb.PapgConfig(max_iters=10**6, gap_norm_tol=-1, infeas_norm_tol=-1, sigma_C=sig)
    s.begin(cfg)
    s.iterate(K)
    stream = s.last_sweep_times() * 1e6
    tot = s.last_timing()[0] / K * 1e6
    s.begin(cfg)
    iso = []
    for _ in range(K):
        s.iterate(1)
        iso.append(s.last_sweep_times()[0] * 1e6)
        time.sleep(0.002)
    iso = np.array(iso)
    # sustained: restart the same early window many times, sampling clocks
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    sus = []
    t0 = time.time()
    while time.time() - t0 < 4.0:
        s.begin(cfg)
        s.iterate(K)
        sus.append(s.last_sweep_times() * 1e6)
    smi.terminate()
    out = smi.communicate()[0]
print("iteration  stream_us  isolated_us  sustained_mean_us")
sus = np.array(sus)
for i in range(K):
    print(f"{i + 1:4d} {stream[i]:9.1f} {iso[i]:9.1f} {sus[:, i].mean():9.1f}")
print(f"step mean (stream) {tot:.1f} us; sweeps 6..{K}: stream {stream[5:].mean():.1f} isolated "
      f"{iso[5:].mean():.1f} sustained {sus[:, 5:].mean():.1f} (runs {len(sus)})")
print("smi samples (sm MHz, W, reasons):")
lines = out.strip().splitlines()
print("\n".join(lines[:: max(1, len(lines) // 40)]))

#!/usr/bin/env python
"""bench.py -- pair-constraint updates/s of the B200 P-APG pair sweep.

Metric (BASELINE.json): pair-constraint updates/s = N^2 * iterations / s, and
time-to-tolerance. A step is one dual iteration of papg_solve over the whole
N x N pair matrix (primal closed form + fused pair sweep + fixed-order reduce
+ control). Workload at 1 GPU: BASELINE config 2 (N = 10000, n = 10,
x ~ U[-1,1]^10, y = max of 20 affine pieces + U[-0.1,0.1] noise, fp64).
With --gpus p > 1 the run is weak-scaled: N = round(1e4 sqrt(p)), so every
GPU sweeps the same 1e8 pairs per iteration over its row block.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation on the host
cores: oracle/_ref (the reference's proj/core sources compiled unmodified, see
oracle/Makefile target `ref`) when it is present, run on a bounded sample of
the same workload (same generator and n, N <= 2000: its sigma_C estimation is
two single-threaded O(N^2 n) passes per power step and cannot be injected);
the oracle port (oracle/cvxreg_oracle.c, all host threads, full N) otherwise.
The line carries both numbers.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_PAIR = 24  # SURVEY 8(d) model: read V, read V', write v (fp64)
READ_BYTES_PER_PAIR = 16  # read V, V' (every pair, every iteration); writes are counted
CONFIGS = {  # BASELINE.json configs
    "cfg1": dict(kind="sqnorm-uniform", N=1000, n=5, noise=0.1, pieces=0),
    "cfg2": dict(kind="maxaffine-uniform", N=10000, n=10, noise=0.1, pieces=20),
    "cfg3": dict(kind="lse-uniform", N=20000, n=20, noise=0.05, pieces=50),
    "cfg4": dict(kind="sqnorm-uniform", N=50000, n=10, noise=0.2, pieces=0),
    "cfg5": dict(kind="maxaffine-uniform", N=100000, n=5, noise=0.1, pieces=10),
}
# sigma_max(C) of each seeded instance (seed 1), for the CPU legs: the device power loop's
# value (profiles/r1n_bench_cfg*.json), which is parity-pinned to the oracle's literal power
# iteration (same step count, sigma within 1e-10: tests/test_gpu_parity.py). The oracle's own
# power iteration is two O(N^2 n) passes per step, too long to run inside a bench.
SIGMA_C = {"cfg1": 75.04526292327877, "cfg2": 289.16619141812674, "cfg3": 532.8884553986682,
           "cfg4": 664.0047049267016, "cfg5": 781.778824412929}
CPU_SAMPLE_S = 30.0  # bound on one CPU sample's work (seconds)
REF_SAMPLE_N = 2000  # N of the compiled reference's bounded sample (sigma_C: ~320 power steps)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip time-to-tolerance and e2e")
    ap.add_argument("--solver", choices=["papg", "alcc", "papg-alcc"], default="papg",
                    help="papg: the north-star P-APG step (default); alcc: one MAPG iteration "
                         "of the standalone ALCC (SURVEY 8f row f1); papg-alcc: one dual "
                         "iteration of the general-K P-APG(ALCC) (row f2)")
    ap.add_argument("--K", type=int, default=2, help="blocks for --solver papg-alcc")
    ap.add_argument("--canonical-blocks", type=int, default=0,
                    help="D > 0: GPU-count-invariant sums over D canonical row blocks "
                         "(cr_set_canonical_blocks; D must be a multiple of --gpus)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak (default): N = N_cfg sqrt(p), fixed pairs per GPU; strong: the "
                         "config's own N on every p (BASELINE cfg 3 and 4 on 1/2/4/8 GPUs, "
                         "cfg 5 on 8)")
    return ap.parse_args()


def workload(name, world, scaling="weak"):
    c = dict(CONFIGS[name])
    if world > 1 and scaling == "weak":
        c["N"] = int(round(c["N"] * math.sqrt(world)))
    return c


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfgname, variant, warmup, steps):
    """DRAM bytes (read + write) per sweep launch, averaged over the launches of this
    command's timed region, from the committed ncu capture of the same command
    (profiles/sweep_traffic.json); None when no capture matches the window."""
    try:
        with open(os.path.join(ROOT, "profiles", "sweep_traffic.json")) as f:
            d = json.load(f)
        e = d.get(f"{cfgname}:{variant}:w{warmup}k{steps}")
        return None if e is None else float(e["dram_bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        time.sleep(0.1)
        self.samples = []
        if self.proc is None:
            return
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def summary(self):
        if not getattr(self, "samples", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def host_mem_available():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_feasible(cfg):
    """BASELINE.md CPU-baseline rule: the oracle holds 4 N^2 doubles (theta1,
    theta1_prev, theta2, C eta); skip when that exceeds 0.8 x MemAvailable."""
    need = 4 * 8 * cfg["N"] ** 2
    avail = host_mem_available()
    return need <= 0.8 * avail, need, avail


def cpu_instance(cfg):
    from oracle import oracle as O

    X, y = O.gen_instance(cfg["kind"], cfg["N"], cfg["n"], cfg["noise"], 1, cfg["pieces"])
    return O, X, O.prepare(X, y)


def cpu_oracle_rate(name, cfg, threads, warm, steps, inst=None):
    """Oracle (CPU restatement of papg.cpp) per-iteration rate on the config: one run of
    warm + steps iterations with sigma_C injected; the timed span is the history's wall
    clock (papg.cpp:220 wall_time_s) from the end of iteration `warm` to the end of
    iteration warm + steps, so setup, warm-up and the final re-solve are outside it.
    Returns (pair-updates/s, seconds of CPU work, sample text, seconds per iteration)."""
    O, X, p = inst or cpu_instance(cfg)
    t0 = time.perf_counter()
    r = O.papg(X, p.ys, max_iters=warm + steps, sigma_C=SIGMA_C[name], gap_norm_tol=-1.0,
               infeas_norm_tol=-1.0, threads=threads, record_history=True, want_theta=False)
    spent = time.perf_counter() - t0
    h = r.history
    t_hi = h[warm + steps - 1, 7]
    t_lo = h[warm - 1, 7] if warm > 0 else 0.0
    per_iter = max(t_hi - t_lo, 1e-9) / steps
    N = cfg["N"]
    sample = (f"{cfg['kind']} N={N} n={cfg['n']}: dual iterations {warm + 1}..{warm + steps} "
              f"of one oracle run (history wall clock), {threads} thread(s), "
              f"{per_iter:.3f} s/iteration")
    return N * N / per_iter, spent, sample, per_iter


def cpu_reference_available():
    from oracle import ref as R

    return R.available()


def cpu_reference_rate(cfg, threads, warm, steps):
    """The REFERENCE's own papg_solve (oracle/_ref: proj/core compiled unmodified, singleton
    blocks through Partition{N, 1}) on a bounded sample of the workload: same generator, n,
    noise and seed at N = min(N_cfg, REF_SAMPLE_N). The timed span is the history's wall clock
    (papg.cpp:220) from the end of iteration `warm` to the end of iteration warm + steps: the
    reference's own sigma_C estimation (papg.cpp:66; it cannot be injected) and the final
    re-solve are outside it. `threads` are the block-pool workers (papg.cpp:69-72); the
    operators are single-threaded (operators.cpp:128-180).
    Returns (pair-updates/s, seconds per iteration, sample text, total seconds)."""
    from oracle import oracle as O
    from oracle import ref as R

    N = min(cfg["N"], REF_SAMPLE_N)
    X, y = O.gen_instance(cfg["kind"], N, cfg["n"], cfg["noise"], 1, cfg["pieces"])
    P = R.prepare(X, y)
    t0 = time.perf_counter()
    r = R.papg(X, P.ys, feas_y=P.feas_y, feas_xi=P.feas_xi, max_iters=warm + steps,
               gap_norm_tol=-1.0, infeas_norm_tol=-1.0, threads=threads, want_theta=False)
    spent = time.perf_counter() - t0
    h = r.history
    t_lo = h[warm - 1, 7] if warm > 0 else 0.0
    per_iter = max(h[warm + steps - 1, 7] - t_lo, 1e-9) / steps
    sample = (f"{cfg['kind']} N={N} n={cfg['n']} (bounded sample of N={cfg['N']}): dual iterations "
              f"{warm + 1}..{warm + steps} of the reference's papg_solve compiled from proj/core "
              f"(history wall clock, its sigma_C estimation excluded), {threads} block-pool "
              f"worker(s), single-threaded operators, {per_iter:.3f} s/iteration, "
              f"{spent:.0f} s in all")
    return N * N / per_iter, per_iter, sample, spent


def cpu_time_to_tolerance(name, cfg, threads, inst=None):
    """Oracle solve of the config to its tolerance (cfg 2: |gap_norm| <= 1e-4, infeas_norm
    <= 0.1), sigma_C injected: measured, not extrapolated."""
    O, X, p = inst or cpu_instance(cfg)
    r = O.papg(X, p.ys, sigma_C=SIGMA_C[name], gap_norm_tol=1e-4, infeas_norm_tol=0.1,
               threads=threads, record_history=False, want_theta=False)
    return {"seconds": r.wall_seconds, "iterations": r.iters, "reason": r.reason,
            "threads": threads, "sigma_C": SIGMA_C[name],
            "includes": "oracle papg loop from zero start to the tolerance and the final re-solve "
                        "(sigma_C injected, not estimated)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = workload(args.config, 1)
    threads = os.cpu_count() or 1
    if cpu_reference_available():
        return run_reference_compiled(args, cfg, threads)
    ok, need, avail = cpu_feasible(cfg)
    if not ok:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"CPU restatement needs {need / 1e9:.0f} GB (4 N^2 doubles) > 0.8 x "
                          f"MemAvailable {avail / 1e9:.0f} GB (BASELINE.md feasibility rule)"}))
        return 0
    W, K = max(args.warmup, 1), max(args.steps, 1)
    inst = cpu_instance(cfg)
    # bound the run to a few minutes: estimate the per-iteration time from one iteration
    # at the configs whose iteration is long (cfg 3, 4); cfg 1 and 2 run W + K as asked
    note = ""
    if cfg["N"] > 10000:
        _, _, _, est = cpu_oracle_rate(args.config, cfg, threads, 0, 1, inst)
        budget = 180.0
        if (W + K) * est > budget:
            K0, W0 = K, W
            W = 1
            K = max(1, int(budget / est) - W)
            note = f"; steps {K0}/warmup {W0} reduced to {K}/{W} to bound the run to ~{budget:.0f} s"
    rate, spent, sample, per = cpu_oracle_rate(args.config, cfg, threads, W, K, inst)
    line = {
        "impl": "reference", "metric": "pair-constraint updates/s", "value": rate,
        "unit": "pair-updates/s", "n_gpus": args.gpus, "steps": K, "warmup": W,
        "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg['kind']} N={cfg['N']} n={cfg['n']}",
                   "N": cfg["N"], "n": cfg["n"], "pairs_per_step": cfg["N"] ** 2,
                   "sigma_C": SIGMA_C[args.config]},
        "cpu_baseline": {"value": rate, "unit": "pair-updates/s", "cores": threads,
                         "kind": "port", "sample": sample + note},
        "e2e": {"value": rate, "unit": "pair-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "oracle/cvxreg_oracle.c (CPU restatement of papg.cpp:136-283, OpenMP rows); "
                "the reference does not build here (Eigen3/vendor absent, alcc.cpp:200-203)",
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference_compiled(args, cfg, threads):
    """--impl reference with oracle/_ref present: the reference's own code (bounded sample),
    and the oracle port on all host threads at the full N beside it when that is feasible."""
    W, K = max(args.warmup, 1), max(args.steps, 1)
    note = ""
    if W + K > 300:  # ~0.11 s per iteration at the sample size: keep the arm within a minute
        K0, W0 = K, W
        W = min(W, 10)
        K = 300 - W
        note = f"; steps {K0}/warmup {W0} reduced to {K}/{W} to bound the run"
    rate, per, sample, _ = cpu_reference_rate(cfg, threads, W, K)
    sample += note
    Ns = min(cfg["N"], REF_SAMPLE_N)
    line = {
        "impl": "reference", "metric": "pair-constraint updates/s", "value": rate,
        "unit": "pair-updates/s", "n_gpus": args.gpus, "steps": K, "warmup": W,
        "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg['kind']} N={cfg['N']} n={cfg['n']}",
                   "N": cfg["N"], "n": cfg["n"], "pairs_per_step": cfg["N"] ** 2,
                   "sample_N": Ns, "sample_pairs_per_step": Ns * Ns},
        "cpu_baseline": {"value": rate, "unit": "pair-updates/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": rate, "unit": "pair-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "oracle/_ref: the reference's proj/core sources compiled unmodified (Eigen calls "
                "served by oracle/eigen_shim, see DESIGN.md section 6); the per-pair rate does not "
                "depend on N (0.0235 G/s at N = 2000, 0.0232 at N = 4000 in the build container)",
    }
    ok, _, _ = cpu_feasible(cfg)
    if ok and cfg["N"] <= 10000:
        pr, _, ps, _ = cpu_oracle_rate(args.config, cfg, threads, 1, 3)
        line["cpu_port_allcores"] = {"value": pr, "unit": "pair-updates/s", "cores": threads,
                                     "kind": "port", "sample": ps}
    print(json.dumps(line), flush=True)
    return 0


def device_rate(crb, name, device, W, K):
    """Iterations W+1 .. W+K of one config on one GPU: pair-updates/s (CUDA events on the
    solver stream) and the sweep's HBM fraction on the bytes it moved."""
    import torch

    c = CONFIGS[name]
    N, n = c["N"], c["n"]
    data = crb.gen_instance(crb.GeneratorSpec(c["kind"], n, N, c["noise"], 1, c["pieces"]))
    prep = crb.prepare_problem(data)
    with crb.DualSolver(prep.data.xs, prep.data.ys, device=device) as s:
        sigma, sig_iters, _ = s.sigma_C()
        s.begin(crb.PapgConfig(max_iters=W + K + 4, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                               sigma_C=sigma, device=device))
        s.iterate(W)
        torch.cuda.synchronize()
        s.sweep_store_count(reset=True)
        done, stopped = s.iterate(K)
        torch.cuda.synchronize()
        dev_s, launches, sweep_s = s.last_timing()
        stores = s.sweep_store_count()
    peaks, _ = measured_peaks()
    moved = READ_BYTES_PER_PAIR * N * N + 8.0 * stores / K
    return {"workload": f"{name}: {c['kind']} N={N} n={n}", "iterations": f"{W + 1}..{W + K}",
            "value": N * N * K / dev_s, "unit": "pair-updates/s", "ms_per_step": dev_s / K * 1e3,
            "sweep_ms": sweep_s / K * 1e3,
            "roofline_frac": moved / (sweep_s / K) / 1e9 / peaks["hbm_gbs"],
            "model_24B_per_pair_frac": 24.0 * N * N / (sweep_s / K) / 1e9 / peaks["hbm_gbs"],
            "sigma_C": sigma, "sigma_power_steps": sig_iters, "gpu_launches": launches}


def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        world = max(world, 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1407_7220_b200 as crb
    from paper_1407_7220_b200.dist import sharded_solver

    cfg = workload(args.config, world, args.scaling)
    N, n = cfg["N"], cfg["n"]
    data = crb.gen_instance(crb.GeneratorSpec(cfg["kind"], n, N, cfg["noise"], 1, cfg["pieces"]))
    prep = crb.prepare_problem(data)

    if world > 1:
        solver = sharded_solver(prep.data.xs, prep.data.ys, group=None, device=local)
    else:
        solver = crb.DualSolver(prep.data.xs, prep.data.ys, device=local)
    sigma, sig_iters, _ = solver.sigma_C()
    W, K = max(args.warmup, 3), args.steps
    pc = crb.PapgConfig(max_iters=W + K + 16, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                        sigma_C=sigma, device=local)
    if args.canonical_blocks > 0:
        solver.set_canonical_blocks(args.canonical_blocks)
    solver.begin(pc)
    solver.iterate(W)

    def barrier():
        if dist is not None:
            dist.barrier()

    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        done0 = solver.iterate(0)[0]
        solver.sweep_store_count(reset=True)
        t_wall0 = time.perf_counter()
        done, stopped = solver.iterate(K)
        t_wall = time.perf_counter() - t_wall0
        torch.cuda.synchronize()
        barrier()
    dev_s, launches, sweep_s = solver.last_timing()
    xchg_s = solver.last_exchange_seconds()
    stores = solver.sweep_store_count()
    assert done - done0 == K and not stopped, (done, done0, stopped)
    t = torch.tensor([dev_s, sweep_s, xchg_s], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_max, sweep_max, xchg_max = float(t[0]), float(t[1]), float(t[2])
    rows = solver.row_end - solver.row_begin
    variant = solver.sweep_variant
    solver.close()

    pairs_step = N * N  # metric unit: N^2 pair-constraint updates per iteration
    value = pairs_step * K / dev_max
    peaks, peak_kind = measured_peaks()
    sweep_avg = sweep_s / K if sweep_s > 0 else None
    # algorithmic bytes per launch: the 16 B/pair reads every iteration needs plus the
    # 8 B stores actually issued (a multiplier equal to the value already in the target
    # buffer is not rewritten; counted by the kernel over the timed launches)
    alg_bytes = READ_BYTES_PER_PAIR * rows * N + 8.0 * stores / K
    achieved = (alg_bytes / sweep_avg / 1e9) if sweep_avg else None
    roofline = {
        "bound": "hbm", "unit": "GB/s", "achieved": achieved, "peak": peaks["hbm_gbs"],
        "frac": (achieved / peaks["hbm_gbs"]) if achieved else None,
        "traffic": ncu_traffic(args.config if world == 1 else "", variant, W, K),
        "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum, mean over the sweep "
                          "launches of the same command's timed region (profiles/sweep_traffic.json)",
        "peak_kind": peak_kind, "kernel": f"sweep ({variant})",
        "algorithmic_bytes_per_launch": alg_bytes,
        "stores_per_launch": stores / K,
        "model_24B_per_pair_frac": (BYTES_PER_PAIR * rows * N / sweep_avg / 1e9 /
                                    peaks["hbm_gbs"]) if sweep_avg else None,
        "sweep_share_of_step": (sweep_s / dev_s) if dev_s > 0 else None,
        "sweep_timing": ("CUDA events on the solver stream around every sweep launch of the "
                         "timed region" if K <= 64 else
                         "CUDA events on the solver stream around every 8th sweep launch of the "
                         "timed region (uniform sample; CRB_SWEEP_EVENTS=1 brackets every launch)"),
        "sweep_launches_timed": K if K <= 64 else (K + 7) // 8,
        # secondary: fp64 flop per pair ~ 4n + 17
        "fp64_tflops": ((4 * n + 17) * rows * N / sweep_avg / 1e12) if sweep_avg else None,
        "note": "SURVEY 8(d) models 24 B per pair (read theta1, theta1_prev, write "
                "theta1_new); the sweep does not rewrite a 32-byte sector whose multipliers "
                "are all unchanged (a sector with a change is written whole), so the "
                "algorithmic bytes are the 16 B/pair reads plus 8 B per multiplier written "
                "(counted on the device); 'model_24B_per_pair_frac' keeps the 24 B view",
    }

    extras = {}
    if not args.no_extras:
        # e2e: the public API call from host arrays, K iterations, sigma estimated inside
        ecfg = crb.PapgConfig(max_iters=K, gap_norm_tol=-1.0, infeas_norm_tol=-1.0, device=local,
                              record_history=False)
        # the inputs of the call live in pinned host memory (bench contract): X and the
        # shifted observations are copied into page-locked buffers the solver uploads from
        xs_pin = torch.empty((N, n), dtype=torch.float64, pin_memory=True)
        ys_pin = torch.empty((N,), dtype=torch.float64, pin_memory=True)
        xs_pin.numpy()[...] = prep.data.xs
        ys_pin.numpy()[...] = prep.data.ys
        prep = crb.PreparedProblem(crb.Dataset(xs_pin.numpy(), ys_pin.numpy()), prep.shift,
                                   prep.feasible, prep.bounds)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world > 1:
            from paper_1407_7220_b200.dist import papg_solve_sharded

            er = papg_solve_sharded(prep, ecfg)
        else:
            er = crb.papg_solve(prep, ecfg, want_dual=False)
        torch.cuda.synchronize()
        barrier()
        e_s = time.perf_counter() - t0
        te = torch.tensor([e_s], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_s = float(te[0])
        h2d = 8 * (N * n + N)  # X and shifted ybar, once per call
        d2h = 8 * (N + N * n)  # fitted y and xi
        extras["e2e"] = {"value": pairs_step * er.report.iters / e_s, "unit": "pair-updates/s",
                         "h2d_bytes_per_step": h2d / K, "d2h_bytes_per_step": d2h / K,
                         "seconds": e_s, "iterations": er.report.iters,
                         "includes": "handle create + H2D of X, ybar from pinned host memory, "
                                     "sigma_C power iteration, K iterations, final re-solve, "
                                     "D2H of (y, xi)"}
        if world == 1 and args.config == "cfg2":
            # time to tolerance: BASELINE cfg 2 runs to |gap_norm| <= 1e-4 (and infeas <= 1e-1)
            # (median of 5 fresh solves: each is ~20 ms, so host-side jitter matters)
            tcfg = crb.PapgConfig(gap_norm_tol=1e-4, device=local)
            runs = []
            for _ in range(5):
                t0 = time.perf_counter()
                tr = crb.papg_solve(prep, tcfg, want_dual=False)
                runs.append((time.perf_counter() - t0, tr))
            runs.sort(key=lambda x: x[0])
            tt, tr = runs[len(runs) // 2]
            extras["time_to_tolerance"] = {
                "seconds": tt, "seconds_min": runs[0][0], "samples": len(runs),
                "iterations": tr.report.iters, "reason": tr.report.reason.name,
                "sigma_seconds": tr.sigma_seconds, "sigma_power_steps": tr.sigma_iters,
                "loop_seconds": tr.loop_seconds, "gap_norm_tol": 1e-4, "infeas_norm_tol": 0.1}
        if world == 1 and args.config == "cfg2":
            # per-iteration rates of the other single-GPU configs at a
            # fixed k, measured by the driver in the same run (early, dense iterations)
            extras["other_configs"] = {c: device_rate(crb, c, local, 5, 10)
                                       for c in ("cfg3", "cfg4")}

    cpu = None
    ok, need, avail = cpu_feasible(cfg)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not ok:
        cpu = {"value": None, "unit": "pair-updates/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"skipped: needs {need / 1e9:.0f} GB > 0.8 x MemAvailable "
                         f"{avail / 1e9:.0f} GB"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and ok:
        threads = os.cpu_count() or 1
        inst = cpu_instance(cfg)
        rate, spent, sample, per = cpu_oracle_rate(args.config, cfg, threads, 1, 3, inst)
        cpu = {"value": rate, "unit": "pair-updates/s", "cores": threads, "kind": "port",
               "sample": sample}
        if cpu_reference_available():
            # the reference's own compiled code on a bounded sample is the baseline; the
            # all-core OpenMP port at the full N stays beside it
            extras["cpu_port_allcores"] = cpu
            rr, _, rs, _ = cpu_reference_rate(cfg, threads, 1, 3)
            cpu = {"value": rr, "unit": "pair-updates/s", "cores": threads, "kind": "reference",
                   "sample": rs}
        # the 1-thread rate beside the all-core one (the reference's
        # operators.cpp:128-180 are single-threaded); one iteration when it fits the bound
        est1 = per * threads
        if 2 * est1 <= CPU_SAMPLE_S or args.config in ("cfg1", "cfg2"):
            r1, _, s1, _ = cpu_oracle_rate(args.config, cfg, 1, 1, 1, inst)
            extras["cpu_baseline_1thread"] = {"value": r1, "unit": "pair-updates/s", "cores": 1,
                                              "kind": "port", "sample": s1}
        if "time_to_tolerance" in extras:
            # measured oracle solve to the same tolerance on all host threads
            extras["time_to_tolerance"]["cpu"] = cpu_time_to_tolerance(args.config, cfg, threads,
                                                                       inst)
        del inst

    if rank == 0:
        line = {
            "metric": "pair-constraint updates/s", "value": value, "unit": "pair-updates/s",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": dev_max / K * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator)",
            "config": {"workload": f"{args.config}: {cfg['kind']} N={N} n={n} "
                                   f"pieces={cfg['pieces']} noise={cfg['noise']}"
                                   + (" (weak scaling N=N_cfg*sqrt(p))" if world > 1 and
                                      args.scaling == "weak" else ""),
                       "N": N, "n": n, "pairs_per_step": pairs_step,
                       "rows_per_gpu": rows, "sweep_variant": variant,
                       "canonical_blocks": args.canonical_blocks,
                       "l2": (f"inputs > L2 (V, V' = {16 * rows * N / 1e9:.3g} GB per GPU), no flush"
                              if 16 * rows * N > 126e6 else
                              f"inputs < L2 (V, V' = {16 * rows * N / 1e6:.3g} MB): L2-resident "
                              "by design, no flush"),
                       "sigma_C": sigma, "sigma_power_steps": sig_iters,
                       "timing": "CUDA events on the solver stream, max over ranks",
                       "wall_s": t_wall},
            "roofline": roofline, "cpu_baseline": cpu, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world > 1:
            # the per-iteration ncclAllReduce of the N(n+2)+4 payload (device time, max over
            # ranks, events around it in the bracketed iterations)
            line["exchange"] = {"seconds": xchg_max, "share_of_step": xchg_max / dev_max,
                                "payload_doubles": N * (n + 2) + 4}
        line.update(extras)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


ALCC_BYTES_PER_PAIR = 8  # theta_k read once per MAPG iteration


def cpu_alcc_rate(cfg, threads, k_lo=1, k_hi=3):
    """Oracle ALCC (alcc.cpp:54-191 restated) per-MAPG-iteration rate: two
    single-outer-step runs with MAPG capped at k_lo and k_hi iterations."""
    from oracle import oracle as O

    X, y = O.gen_instance(cfg["kind"], cfg["N"], cfg["n"], cfg["noise"], 1, cfg["pieces"])
    p = O.prepare(X, y)
    kw = dict(gamma=p.gamma, Bbar_y=p.Bbar_y, Bbar_xi=p.Bbar_xi, warm_y=p.feas_y,
              warm_xi=p.feas_xi, sigma_A1=100.0, sigma_A2=100.0, max_outer=1,
              alpha1_scale=1e-30, infeas_norm_tol=-1.0, threads=threads, record_history=False)
    t0 = time.perf_counter()
    a = O.alcc(X, p.ys, mapg_cap=k_lo, **kw)
    b = O.alcc(X, p.ys, mapg_cap=k_hi, **kw)
    spent = time.perf_counter() - t0
    per_iter = max(b.wall_seconds - a.wall_seconds, 1e-9) / max(b.mapg_iters_total -
                                                                a.mapg_iters_total, 1)
    N = cfg["N"]
    sample = (f"{cfg['kind']} N={N} n={cfg['n']}: oracle ALCC, one outer step with MAPG capped at "
              f"{k_lo} and {k_hi} iterations, {threads} thread(s), {per_iter:.3f} s/MAPG iteration")
    return N * N / per_iter, spent, sample


def run_alcc_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    cfg = workload(args.config, 1)
    threads = os.cpu_count() or 1
    need = 7 * 8 * cfg["N"] ** 2
    if need > 0.8 * host_mem_available():
        print(json.dumps({"impl": "reference", "unavailable": "ALCC oracle needs 7 N^2 doubles"}))
        return 0
    rate, spent, sample = cpu_alcc_rate(cfg, threads)
    line = {
        "impl": "reference", "metric": "MAPG pair evaluations/s", "value": rate,
        "unit": "pair-evals/s", "n_gpus": args.gpus, "steps": 2, "warmup": 1,
        "ms_per_step": cfg["N"] ** 2 / rate * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"alcc {args.config}: {cfg['kind']} N={cfg['N']} n={cfg['n']}",
                   "N": cfg["N"], "n": cfg["n"], "solver": "alcc"},
        "cpu_baseline": {"value": rate, "unit": "pair-evals/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "pair-evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_alcc_ours(args):
    """One MAPG iteration of the standalone ALCC is the step (penalty sweep +
    reduce + gradient + projection/momentum kernels, device-resident)."""
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(local)
    import paper_1407_7220_b200 as crb

    cfg = workload(args.config, 1)
    N, n = cfg["N"], cfg["n"]
    data = crb.gen_instance(crb.GeneratorSpec(cfg["kind"], n, N, cfg["noise"], 1, cfg["pieces"]))
    prep = crb.prepare_problem(data)
    W, K = max(args.warmup, 3), max(args.steps, 10)
    with crb.DualSolver(prep.data.xs, prep.data.ys, prep.bounds.gamma, local) as s:
        t0 = time.perf_counter()
        s1 = s.sigma_A(1)
        s2 = s.sigma_A(2)
        sig_s = time.perf_counter() - t0
        # alpha1_scale -> 0: the displacement test never fires, MAPG runs exactly cap steps
        base = dict(max_outer=1, alpha1_scale=1e-30, infeas_norm_tol=-1.0, sigma_A1=s1[0],
                    sigma_A2=s2[0], record_history=False)
        s.alcc(crb.AlccConfig(mapg_cap=W, **base), prep.bounds, prep.feasible)
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            res, *_ = s.alcc(crb.AlccConfig(mapg_cap=K, **base), prep.bounds, prep.feasible)
            torch.cuda.synchronize()
        sweep_s = s.time_penalty_sweep(20)
        variant = s.sweep_variant
    iters = int(res.mapg_iters_total)
    assert iters == K, (iters, K)
    dev = res.mapg_seconds
    value = N * N * iters / dev
    peaks, peak_kind = measured_peaks()
    achieved = ALCC_BYTES_PER_PAIR * N * N / sweep_s / 1e9
    roofline = {"bound": "hbm", "unit": "GB/s", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_kind": peak_kind,
                "kernel": f"penalty sweep ({variant})",
                "algorithmic_bytes_per_launch": ALCC_BYTES_PER_PAIR * N * N,
                "sweep_share_of_step": sweep_s * iters / dev,
                "note": "8 B/pair leaves the sweep FP64-issue bound, not HBM bound"}
    extras = {}
    if not args.no_extras:
        ecfg = crb.AlccConfig(mapg_cap=K, max_outer=1, alpha1_scale=1e-30, infeas_norm_tol=-1.0,
                              record_history=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        er = crb.alcc_solve(prep, ecfg, want_multiplier=False)
        e_s = time.perf_counter() - t0
        extras["e2e"] = {"value": N * N * er.mapg_iters_total / e_s, "unit": "pair-evals/s",
                         "h2d_bytes_per_step": 8 * (N * n + N) * 2 / K,
                         "d2h_bytes_per_step": 8 * (N + N * n) / K, "seconds": e_s,
                         "iterations": er.mapg_iters_total,
                         "includes": "handle create + H2D, sigma(A1), sigma(A2), one outer step "
                                     "of K MAPG iterations, D2H of (y, xi)"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline and 7 * 8 * N * N <= 0.8 * host_mem_available():
        threads = os.cpu_count() or 1
        rate, spent, sample = cpu_alcc_rate(cfg, threads)
        cpu = {"value": rate, "unit": "pair-evals/s", "cores": threads, "kind": "port",
               "sample": sample}
    line = {
        "metric": "MAPG pair evaluations/s", "value": value, "unit": "pair-evals/s", "n_gpus": 1,
        "steps": K, "warmup": W, "ms_per_step": dev / iters * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator)",
        "config": {"workload": f"alcc {args.config}: {cfg['kind']} N={N} n={n} (one outer step, "
                               f"K MAPG iterations)", "N": N, "n": n, "solver": "alcc",
                   "sweep_variant": variant, "sigma_A": [s1[0], s2[0]],
                   "sigma_power_steps": [s1[1], s2[1]], "sigma_seconds": sig_s,
                   "l2": f"theta ({8 * N * N / 1e9:.3g} GB) " + ("> L2, no flush" if 8 * N * N > 126e6
                                                                        else "< L2, no flush"),
                   "timing": "CUDA events around the MAPG graph launches"},
        "roofline": roofline, "cpu_baseline": cpu, "gpu_launches": int(res.launches),
        "clocks": clk.summary(),
    }
    line.update(extras)
    print(json.dumps(line), flush=True)
    return 0


# f2 workload: the reference's default solver (K = 2) with a bounded inner ALCC so a
# step is a fixed amount of work on both arms (identical inner iteration counts)
GEN_INNER = dict(max_outer=5, mapg_cap=200)


def run_general(args, impl):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    cfg = workload(args.config, 1)
    N, n, K = cfg["N"], cfg["n"], args.K
    K_steps = max(1, min(args.steps, 5)) if impl == "reference" else max(1, args.steps)
    line_cfg = {"workload": f"papg-alcc {args.config}: {cfg['kind']} N={N} n={n} K={K} "
                            f"(inner ALCC max_outer={GEN_INNER['max_outer']}, "
                            f"mapg_cap={GEN_INNER['mapg_cap']})",
                "N": N, "n": n, "K": K, "solver": "papg-alcc"}
    if impl == "reference":
        from oracle import oracle as O
        X, y = O.gen_instance(cfg["kind"], N, n, cfg["noise"], 1, cfg["pieces"])
        p = O.prepare(X, y)
        threads = os.cpu_count() or 1
        sig = SIGMA_C.get(args.config, 300.0) if K == N else 300.0  # cost does not depend on it
        kw = dict(inner=GEN_INNER, sigma_C=sig, gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                  record_history=False, inner_threads=threads)
        a = O.papg_k(X, p.ys, K, p.feas_y, p.feas_xi, max_iters=1, **kw)
        b = O.papg_k(X, p.ys, K, p.feas_y, p.feas_xi, max_iters=1 + K_steps, **kw)
        per = max(b.wall_seconds - a.wall_seconds, 1e-9) / K_steps
        rate = 1.0 / per
        sample = (f"oracle papg_k (papg.cpp + alcc.cpp restated), runs of 1 and {1 + K_steps} "
                  f"dual iterations, blocks sequential, {threads} thread(s) per block solve, "
                  f"{per:.3f} s/iteration")
        line = {"impl": "reference", "metric": "P-APG(ALCC) dual iterations/s", "value": rate,
                "unit": "iterations/s", "n_gpus": args.gpus, "steps": K_steps, "warmup": 1,
                "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": line_cfg,
                "cpu_baseline": {"value": rate, "unit": "iterations/s", "cores": threads,
                                 "kind": "port", "sample": sample},
                "e2e": {"value": rate, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    import paper_1407_7220_b200 as crb
    data = crb.gen_instance(crb.GeneratorSpec(cfg["kind"], n, N, cfg["noise"], 1, cfg["pieces"]))
    prep = crb.prepare_problem(data)
    inner = crb.AlccConfig(**GEN_INNER)
    W = max(args.warmup, 3) if args.warmup else 3
    with crb.DualSolver(prep.data.xs, prep.data.ys, prep.bounds.gamma, local) as s:
        s.set_partition(K, prep.feasible, inner)
        sig = s.sigma_C()
        pc = crb.PapgConfig(K=K, inner=inner, max_iters=W + K_steps + 4, gap_norm_tol=-1.0,
                            infeas_norm_tol=-1.0, sigma_C=sig[0], device=local)
        s.begin(pc)
        s.iterate(W)
        st0 = s.partition_stats()
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            done, stopped = s.iterate(K_steps)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        st1 = s.partition_stats()
        sec, launches, sweep_s = s.last_timing()
    inner_it = st1["inner_iters"] - st0["inner_iters"]
    nb = N // K
    pairs = K_steps * N * (N - nb) + inner_it * nb * nb
    extras = {}
    if not args.no_extras:
        # e2e: papg_solve from host arrays (partition setup, sigma, K_steps iterations,
        # final block re-solve, D2H of eta)
        ecfg = crb.PapgConfig(K=K, inner=inner, max_iters=K_steps, gap_norm_tol=-1.0,
                              infeas_norm_tol=-1.0, record_history=False, device=local)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        er = crb.papg_solve(prep, ecfg, want_dual=False)
        e_s = time.perf_counter() - t0
        extras["e2e"] = {"value": er.report.iters / e_s, "unit": "iterations/s",
                         "h2d_bytes_per_step": 8 * (N * n + N) * 2 / K_steps,
                         "d2h_bytes_per_step": 8 * (N + N * n) / K_steps, "seconds": e_s,
                         "includes": "handle + partition setup (block sigmas), sigma_C, the "
                                     "dual iterations, final block re-solve, D2H of eta"}
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import oracle as O
        X, y = O.gen_instance(cfg["kind"], N, n, cfg["noise"], 1, cfg["pieces"])
        p = O.prepare(X, y)
        threads = os.cpu_count() or 1
        kw = dict(inner=GEN_INNER, sigma_C=sig[0], gap_norm_tol=-1.0, infeas_norm_tol=-1.0,
                  record_history=False, inner_threads=threads)
        a = O.papg_k(X, p.ys, K, p.feas_y, p.feas_xi, max_iters=1, **kw)
        b = O.papg_k(X, p.ys, K, p.feas_y, p.feas_xi, max_iters=2, **kw)
        per = max(b.wall_seconds - a.wall_seconds, 1e-9)
        cpu = {"value": 1.0 / per, "unit": "iterations/s", "cores": threads, "kind": "port",
               "sample": f"oracle papg_k, dual iteration 2 (runs of 1 and 2), {threads} "
                         f"thread(s) per block solve, {per:.3f} s"}
    line = {"metric": "P-APG(ALCC) dual iterations/s", "value": K_steps / wall,
            "unit": "iterations/s", "n_gpus": 1, "steps": K_steps, "warmup": W,
            "ms_per_step": wall / K_steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE generator)",
            "config": dict(line_cfg, sigma_C=sig[0], inner_mapg_iterations=inner_it,
                           pair_evaluations=pairs, pair_evals_per_s=pairs / wall,
                           cross_sweep_seconds=sweep_s,
                           timing="host wall clock around device-synchronised iterations "
                                  "(host-driven block solves)"),
            "roofline": None, "cpu_baseline": cpu, "gpu_launches": None,
            "clocks": clk.summary()}
    line.update(extras)
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.solver == "papg-alcc":
        return run_general(args, args.impl)
    if args.solver == "alcc":
        return run_alcc_reference(args) if args.impl == "reference" else run_alcc_ours(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

"""Summarise an ncu report: SASS opcode mix, stall reasons, key raw metrics."""
import collections, csv, subprocess, sys

rep = sys.argv[1]
pairs = float(sys.argv[2]) if len(sys.argv) > 2 else 0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src))
hdr = rows[1]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
ops, stall, tot = collections.Counter(), collections.Counter(), 0
for r in rows[2:]:
    try:
        e = int(r[iE] or 0)
    except ValueError:
        continue
    t = r[iS].strip().split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] += e
    tot += e
    try:
        stall[op] += int(r[iW] or 0)
    except ValueError:
        pass
print(f"warp instructions {tot}" + (f"  thread-instr/pair {tot*32/pairs:.1f}" if pairs else ""))
for op, c in ops.most_common(20):
    print(f"  {op:10s} {c:12d} {c/tot*100:5.1f}%  stall-samples {stall[op]}")
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                     capture_output=True, text=True).stdout.splitlines()))
h, v = raw[0], raw[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second"]
for i, name in enumerate(h):
    if name in keys:
        print(f"  {name} = {v[i]} {raw[1][i]}")
st = []
for i, name in enumerate(h):
    if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"):
        try:
            st.append((float(v[i]), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
print("  stalls:", ", ".join(f"{n}={int(x)}" for x, n in sorted(st, reverse=True)[:8]))

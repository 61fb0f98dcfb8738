"""Writes profiles/<tag>_* from gpurun_out captures (launch list + one ncu --set full).

  python scripts/summarize_profiles.py <tag> <config> <variant> <launches.csv> <sweep.ncu-rep> <steps>
"""
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, cfg, variant, launches, rep, steps = sys.argv[1:7]
steps = int(steps)
prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)

rows = list(csv.reader(open(launches)))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hdr]
iN, iV = h.index("Kernel Name"), h.index("Metric Value")
ks = [(re.sub(r"\(.*", "", r[iN]).split("::")[-1], float(r[iV])) for r in rows[hdr + 1:] if len(r) > iV]
lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised), {len(ks)} launches",
         "kernel,count,total_us,avg_us"]
tot, cnt = collections.Counter(), collections.Counter()
for n, v in ks:
    tot[n] += v
    cnt[n] += 1
for n in tot:
    lines.append(f"{n},{cnt[n]},{tot[n] / 1e3:.1f},{tot[n] / cnt[n] / 1e3:.2f}")
per_iter = 3
last = ks[-steps * per_iter:]
share = collections.Counter()
for n, v in last:
    share[n] += v
s = sum(share.values())
lines.append(f"# timed region (last {steps} iterations): step {s / steps / 1e3:.1f} us")
for n, v in share.items():
    lines.append(f"# share {n}: {v / s:.4f}")
open(os.path.join(prof, f"{tag}_launches.csv"), "w").write("\n".join(lines) + "\n")

summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                      capture_output=True, text=True).stdout
open(os.path.join(prof, f"{tag}_sweep_ncu.txt"), "w").write(
    f"# ncu --set full --clock-control none, one {variant} sweep launch of {cfg}\n" + summ)
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                     capture_output=True, text=True).stdout.splitlines()))
m = dict(zip(raw[0], raw[2]))
units = dict(zip(raw[0], raw[1]))


def val(name):
    v = float(m[name].replace(",", ""))
    u = units[name]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
             "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1)
    return v * scale


traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
path = os.path.join(prof, "sweep_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[f"{cfg}:{variant}"] = {"dram_bytes_per_launch": traffic,
                         "duration_s": val("gpu__time_duration.sum"), "source": f"{tag}_sweep_ncu.txt"}
json.dump(d, open(path, "w"), indent=1)
print(open(os.path.join(prof, f"{tag}_launches.csv")).read())
print(summ)

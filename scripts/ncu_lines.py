"""Per CUDA source line: warp instructions executed and stall samples, from an
ncu report (--import-source, -lineinfo). python scripts/ncu_lines.py rep [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
f = None
rows = []
hdr = None
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    if ie or st:
        rows.append((f, int(r[0]), r[1].strip()[:70], ie, st))
tot_i = sum(x[3] for x in rows)
tot_s = sum(x[4] for x in rows)
print(f"total warp instr {tot_i}, stall samples {tot_s}")
print("-- by instructions")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{x[0]:>14s}:{x[1]:<5d} {x[3] / tot_i * 100:5.1f}% instr {x[4] / tot_s * 100:5.1f}% stall  {x[2]}")
print("-- by stall samples")
for x in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{x[0]:>14s}:{x[1]:<5d} {x[3] / tot_i * 100:5.1f}% instr {x[4] / tot_s * 100:5.1f}% stall  {x[2]}")

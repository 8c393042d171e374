"""Stall samples and executed instructions per CUDA source line from an ncu report (cuda,sass view;
needs -lineinfo and --import-source). usage: ncu_lines.py REPORT [TOP]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = {}
fname = "?"
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        n = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0, 0, r[1].strip()[:90]])
    a[0] += s
    a[1] += n
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot}  warp-instructions {toti}")
for (f, ln), (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}% stall {100 * n / toti:5.1f}% instr  {f}:{ln}  {src}")

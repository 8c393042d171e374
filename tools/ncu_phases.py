"""Split a kernel's SASS (ncu source page) into phases at BAR instructions and report, per phase,
stall samples by reason and the instruction mix. usage: ncu_phases.py REPORT KERNEL_REGEX [SKIP]"""
import collections
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
print(rows[0][1][:110])
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
phases = []
cur = {"n": 0, "s": collections.Counter(), "ops": collections.Counter(), "inst": 0, "first": None}
total = 0
for r in rows[2:]:
    if len(r) < len(hdr) or not r[col["Instructions Executed"]].strip().isdigit():
        continue
    src = r[col["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    opb = op.split(".")[0]
    if cur["first"] is None:
        cur["first"] = src[:40]
    for h in reasons:
        v = int(r[col[h]] or 0)
        cur["s"][h[6:]] += v
        total += v
    n = int(r[col["Instructions Executed"]] or 0)
    cur["inst"] += n
    cur["ops"][opb] += n
    if opb == "BAR":
        phases.append(cur)
        cur = {"n": 0, "s": collections.Counter(), "ops": collections.Counter(), "inst": 0, "first": None}
phases.append(cur)
for i, p in enumerate(phases):
    st = sum(p["s"].values())
    if st == 0 and p["inst"] == 0:
        continue
    top = ", ".join(f"{k}:{100 * v / max(total, 1):.1f}" for k, v in p["s"].most_common(4) if v)
    ops = ", ".join(f"{k}:{v // 1000}k" for k, v in p["ops"].most_common(5))
    print(f"phase {i:2d} stall {100 * st / max(total, 1):5.1f}%  [{top}]  ops[{ops}]  starts '{p['first']}'")

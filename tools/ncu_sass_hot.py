"""Aggregate an ncu SASS source page: stall samples and executed instructions by opcode, plus the
hottest instructions. usage: ncu_sass_hot.py REPORT KERNEL_REGEX [SKIP]"""
import collections
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
print(rows[0][1][:120])
hdr = rows[1]
iS, iI, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
by_op = collections.Counter()
by_op_i = collections.Counter()
data = []
for r in rows[2:]:
    try:
        s, n = int(r[iS] or 0), int(r[iI] or 0)
    except (ValueError, IndexError):
        continue
    op = r[iSrc].split()[0] if r[iSrc].split() else "?"
    if op.startswith("@"):
        op = r[iSrc].split()[1]
    op = op.split(".")[0]
    by_op[op] += s
    by_op_i[op] += n
    data.append((s, n, r[iSrc].strip()[:90]))
tot = sum(by_op.values()) or 1
toti = sum(by_op_i.values()) or 1
print(f"samples {tot} warp-instructions {toti}")
for op, s in by_op.most_common(18):
    print(f"  {op:10s} stall {100 * s / tot:5.1f}%   instr {100 * by_op_i[op] / toti:5.1f}%")
print("hottest:")
for s, n, src in sorted(data, reverse=True)[:12]:
    print(f"  {100 * s / tot:5.1f}% {src}")

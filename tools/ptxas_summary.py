"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spills (reads stdin)."""
import re, subprocess, sys
cur = None
mangled = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = mangled = m.group(1)
        try:
            cur = subprocess.run(["c++filt"], input=cur, capture_output=True, text=True).stdout.strip()
        except Exception:
            pass
        rows[cur] = {}
        continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:   # non-entry functions have their own property blocks: do not charge them to the kernel
        prop = m.group(1)
        cur = cur if cur is not None and mangled == prop else None
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows[cur]["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    short = re.sub(r"\(.*", "", k)
    print(f"{v.get('regs', '?'):>4} regs {v.get('spill', 0):>5} spill  {short}")

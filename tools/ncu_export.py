"""Export per-kernel ncu metrics (one --set full capture) to a JSON summary under profiles/.
usage: python tools/ncu_export.py OUT.json REPORT_OR_RAW_CSV [...]"""
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time_ms",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "launch__registers_per_thread": "registers",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sass__inst_executed_register_spilling": "spill_instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3, "ns": 1e-6, "Ghz": 1e9,
        "Mhz": 1e6, "hz": 1.0}


def main(out, *reps):
    """reps: .ncu-rep files or their `--page raw --csv` exports; all launches go into one summary."""
    res = []
    for rep in reps:
        res += launches(rep)
    with open(out, "w") as f:
        json.dump({"reports": list(reps), "launches": res}, f, indent=1)
    for d in res:
        print(f"{d['kernel']:40s} {d.get('time_ms', 0):8.4f} ms  dram {d.get('dram_bytes', 0) / 1e6:9.1f} MB")


def launches(rep):
    if rep.endswith(".csv"):
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, short in KEYS.items():
            if k not in hdr:
                continue
            i = hdr.index(k)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            d[short] = v * UNIT.get(units[i].strip(), 1.0)
        if "dram_read_bytes" in d and "dram_write_bytes" in d:
            d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        res.append(d)
    return res


if __name__ == "__main__":
    main(*sys.argv[1:])

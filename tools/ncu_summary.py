"""Summarise an ncu report: per kernel launch, the metrics the B200 recipe asks for."""
import csv
import subprocess
import sys

WANT = [
    ("Kernel Name", "kernel"), ("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("launch__registers_per_thread", "regs"), ("launch__block_size", "block"), ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"), ("launch__occupancy_limit_shared_mem", "occ_lim_smem"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64pipe%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fmapipe%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("sass__inst_executed_register_spilling", "spill_inst"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_longsb"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_shortsb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall_mio"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall_math"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall_notsel"),
    ("sm__cycles_elapsed.avg.per_second", "clk"),
]


def main(rep, pattern=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = [(hdr.index(k) if k in hdr else -1, short) for k, short in WANT]
    for r in rows[2:]:
        if pattern and pattern not in r[hdr.index("Kernel Name")]:
            continue
        parts = []
        for i, short in idx:
            if i < 0:
                continue
            v = r[i]
            if short == "kernel":
                v = v.split("(")[0].replace("void ", "")
            parts.append(f"{short}={v}{'' if short == 'kernel' else units[i].replace(' ', '')}")
        print(" | ".join(parts))


if __name__ == "__main__":
    main(*sys.argv[1:])

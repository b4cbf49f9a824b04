"""Summarise an ncu report: key throughput metrics and warp-stall breakdown.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-index]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
    "launch__block_size", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "lts__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]
for r in rows[2:]:
    print("-" * 60)
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k:70s} {r[i]} {u[i]}")
    for i in range(len(h)):  # FP64 tensor (DMMA) pipe, when the kernel uses it
        if "dmma" in h[i] and "pct_of_peak_sustained_active" in h[i] and r[i] not in ("", "n/a"):
            print(f"{h[i]:70s} {r[i]} {u[i]}")
    st = [(h[i], float(r[i].replace(",", ""))) for i in range(len(h))
          if re.match(r"smsp__pcsamp_warps_issue_stalled_\w+$", h[i]) and r[i] not in ("", "n/a")]
    tot = sum(v for _, v in st) or 1
    for k, v in sorted(st, key=lambda x: -x[1])[:10]:
        print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {v / tot:6.1%}")

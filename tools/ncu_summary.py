"""Summarise an ncu --set full report of the back-projection kernel (markdown to stdout).

    python tools/ncu_summary.py gpurun_out/<report>.ncu-rep [updates]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
updates = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = open(rep).read() if rep.endswith(".csv") else subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
M = {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def g(name):
    v, u = M.get(name, ("n/a", ""))
    return v, u


keys = [
    ("Kernel", "Kernel Name"),
    ("Duration", "gpu__time_duration.sum"),
    ("SM clock", "sm__cycles_elapsed.avg.per_second"),
    ("Registers/thread", "launch__registers_per_thread"),
    ("Block size", "launch__block_size"),
    ("Grid size", "launch__grid_size"),
    ("Dynamic smem/block", "launch__shared_mem_per_block_dynamic"),
    ("Warps active/SM (achieved)", "sm__warps_active.avg.per_cycle_active"),
    ("Issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("Executed instructions (warp)", "smsp__inst_executed.sum"),
    ("FMA pipe cycles active %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("FMA-heavy pipe cycles active %", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("ALU pipe active %", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    ("LSU inst executed %", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("Shared wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("Shared bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("L1/shared data-pipe utilisation %", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    ("DRAM read bytes", "dram__bytes_read.sum"),
    ("DRAM write bytes", "dram__bytes_write.sum"),
    ("L2 throughput %", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed"),
    ("TMA pipe active %", "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active"),
]
print(f"# ncu summary: `{rep.split('/')[-1]}`\n")
print("| metric | value |\n|---|---|")
for label, k in keys:
    v, u = g(k)
    print(f"| {label} (`{k}`) | {v} {u} |")
inst = g("smsp__inst_executed.sum")[0]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
try:
    dram = sum(float(g(k)[0]) * SCALE.get(g(k)[1], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    print(f"| DRAM traffic per launch (read + write) | {dram / 1e6:.1f} MB |")
    if updates:
        print(f"| warp instructions per 32 updates | {float(inst) * 32 / updates:.1f} |")
except ValueError:
    pass
stalls = []
for h, (v, u) in M.items():
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            stalls.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("\nTop stall reasons (warps per issued instruction):\n")
for v, h in sorted(stalls, reverse=True)[:8]:
    print(f"- {h}: {v:.2f}")

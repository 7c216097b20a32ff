"""Summarise an ncu --set full report into markdown (development helper).
usage: python tools/ncu_summary.py report.ncu-rep [title] > profiles/xxx.md"""
import csv, subprocess, sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
units = {}
if len(rows) > 1:
    units = dict(zip(h, rows[1]))
print(f"# {title}\n")
print("ncu --set full --clock-control none (one launch per kernel; cold cache, serialised).\n")
for row in rows[2:]:
    d = dict(zip(h, row))
    print(f"## {d['Kernel Name']}\n")
    for k, name in want:
        if k in d:
            print(f"- {name}: {d[k]} {units.get(k, '')}".rstrip())
    stalls = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print("- top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:5]))
    print()

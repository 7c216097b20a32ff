"""Summarise an ncu --set full report (one entry per captured launch) as markdown:
time, DRAM bytes and % of peak, pipe activity, occupancy, registers, top stalls.

    python tools/ncu_summary.py report.ncu-rep [title]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("time (us)", "gpu__time_duration.sum", 1e-3),
    ("DRAM read (MB)", "dram__bytes_read.sum", 1e-6),
    ("DRAM write (MB)", "dram__bytes_write.sum", 1e-6),
    ("DRAM % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("DMMA pipe %", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("registers", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
]


def units(row, h, key):
    try:
        return row[h.index(key)]
    except ValueError:
        return None


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, unit_row = rows[0], rows[1]
    print(f"# {title}\n\nncu --set full --clock-control none (one launch per kernel; cold cache, serialised).\n")
    for row in rows[2:]:
        print(f"## {row[h.index('Kernel Name')]}\n")
        for label, key, scale in KEYS:
            v = units(row, h, key)
            if v is None or v == "":
                continue
            u = unit_row[h.index(key)]
            try:
                x = float(v.replace(",", ""))
                if key == "gpu__time_duration.sum":
                    x = x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)
                    print(f"- {label}: {x:.1f}")
                    continue
                if key.startswith("dram__bytes"):
                    x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
                    print(f"- {label}: {x:.1f}")
                    continue
                print(f"- {label}: {x:g}")
            except ValueError:
                print(f"- {label}: {v}")
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(row[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        if st:
            print("- top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:5]))
        print()


if __name__ == "__main__":
    main()

"""Executed-instruction mix by opcode from an ncu report (development helper).
usage: python tools/ncu_sass_mix.py report.ncu-rep [kernel_index]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
kernels = []; cur = None; h = None
for x in csv.reader(out.splitlines()):
    if x and x[0] == "Kernel Name":
        cur = [x[1], []]; kernels.append(cur); h = None; continue
    if h is None and x and x[0] == "Address":
        h = x; continue
    if cur is not None and h is not None and len(x) == len(h):
        cur[1].append(x)
name, rows = kernels[kidx]
ei = h.index("Instructions Executed")
c = collections.Counter()
for x in rows:
    op = x[1].split()
    if op and op[0].startswith("@"): op = op[1:]
    c[op[0].split(".")[0] if op else "?"] += int(x[ei] or 0)
tot = sum(c.values())
print(name, "warp instructions", tot)
for k, v in c.most_common(25): print(f"  {k:10s} {v:12d} {v/tot:6.1%}")

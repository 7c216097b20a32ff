"""Top SASS lines by warp-stall samples from an ncu report (development helper).
usage: python tools/ncu_sass_hot.py report.ncu-rep [kernel_index] [n]"""
import csv, subprocess, sys
rep = sys.argv[1]; kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0; top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines())
kernels = []; cur = None; h = None
for x in r:
    if x and x[0] == "Kernel Name":
        cur = [x[1], []]; kernels.append(cur); h = None; continue
    if h is None and x and x[0] == "Address":
        h = x; continue
    if cur is not None and h is not None and len(x) == len(h):
        cur[1].append(x)
name, rows = kernels[kidx]
si = h.index("Warp Stall Sampling (All Samples)")
cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(int(x[si]) for x in rows)
agg = {}
for x in rows:
    for i in cols:
        agg[h[i]] = agg.get(h[i], 0) + int(x[i] or 0)
print(name, "samples", tot, "instructions", len(rows))
print("  ", ", ".join(f"{k[6:]}={v/tot:.1%}" for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
for i, x in sorted(enumerate(rows), key=lambda t: -int(t[1][si]))[:top]:
    reasons = sorted(((int(x[c] or 0), h[c][6:]) for c in cols), reverse=True)[:2]
    print(f"{i:6d} {int(x[si]):6d} {x[1][:60]:60s} {reasons}")

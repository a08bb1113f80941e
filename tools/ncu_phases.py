"""Split a kernel's ncu warp-stall samples into phases delimited by BAR.SYNC
(SASS order).  usage: python tools/ncu_phases.py report.ncu-rep kernel_regex"""
import csv
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
ie = hdr.index("Instructions Executed")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(x):
    try:
        return int(float(x))
    except ValueError:
        return 0


phase, acc, ins, reasons = 0, defaultdict(int), defaultdict(int), defaultdict(lambda: defaultdict(int))
for r in data:
    acc[phase] += num(r[si])
    ins[phase] += num(r[ie])
    for c in cols:
        reasons[phase][c] += num(r[hdr.index(c)])
    if "BAR.SYNC" in r[src] or "EXIT" in r[src] and phase == 0:
        phase += 1
tot = sum(acc.values())
for p in sorted(acc):
    top = sorted(reasons[p].items(), key=lambda x: -x[1])[:3]
    print(f"phase {p:2d}: samples {acc[p]:7d} ({100 * acc[p] / max(tot, 1):5.1f}%)  warp-inst {ins[p]:10d}  ",
          ", ".join(f"{k[6:]}={v}" for k, v in top))

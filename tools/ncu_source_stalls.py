"""Aggregate ncu source-page (SASS) warp-stall samples by opcode.
usage: python tools/ncu_source_stalls.py report.ncu-rep kernel_regex"""
import csv
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(num(r[si]) for r in data if len(r) == len(hdr))
agg = defaultdict(lambda: defaultdict(int))
cnt = defaultdict(int)
data = [r for r in data if len(r) == len(hdr)]
for r in data:
    toks = r[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    cnt[op] += num(r[si])
    for c in cols:
        agg[op][c] += num(r[hdr.index(c)])
print("total samples", tot)
for op, v in sorted(cnt.items(), key=lambda x: -x[1])[:14]:
    top = sorted(agg[op].items(), key=lambda x: -x[1])[:4]
    print(f"{op:12s} {v:7d} {100 * v / max(tot, 1):5.1f}%  ", ", ".join(f"{k[6:]}={w}" for k, w in top))

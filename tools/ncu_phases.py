"""Split a kernel's ncu source-page rows (SASS order) into phases delimited by
BAR.SYNC / EXIT: warp-stall samples, executed warp instructions and the opcode
mix per phase, then the kernel's executed opcode totals.  The source page
lists every SASS row once per inlined view, so rows are de-duplicated by
address.  usage: python tools/ncu_phases.py report.ncu-rep kernel_regex"""
import csv
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
print(rows[0][1] if len(rows[0]) > 1 else rows[0])
hdr = rows[1]
A, S = hdr.index("Address"), hdr.index("Source")
SI, IE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [(h, hdr.index(h)) for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
seen, data = set(), []
for r in rows[2:]:
    if len(r) != len(hdr) or r[A] == "Address" or r[A] in seen:
        continue
    seen.add(r[A])
    data.append(r)


def num(x):
    try:
        return int(float(x))
    except ValueError:
        return 0


tot = sum(num(r[SI]) for r in data) or 1
ti = sum(num(r[IE]) for r in data) or 1
print(f"sass rows {len(data)}  stall samples {tot}  warp instructions {ti}")
ph, acc, ins, n, ops, why, allops = 0, 0, 0, 0, Counter(), Counter(), Counter()
for r in data:
    e = num(r[IE])
    acc += num(r[SI])
    ins += e
    n += 1
    t = r[S].split()
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += e
    allops[op] += e
    for h, i in stall_cols:
        why[h[6:]] += num(r[i])
    if "BAR.SYNC" in r[S] or "EXIT" in r[S]:
        if acc or ins:
            print(f"phase {ph:2d}: rows {n:5d}  samples {acc:6d} ({100 * acc / tot:5.1f}%)  inst {ins:10d} "
                  f"({100 * ins / ti:5.1f}%)  stalls " + ", ".join(f"{k}={v}" for k, v in why.most_common(3)) +
                  "  ops " + ", ".join(f"{k}={v / 1e6:.2f}M" for k, v in ops.most_common(6)))
        ph, acc, ins, n, ops, why = ph + 1, 0, 0, 0, Counter(), Counter()
print("executed opcodes: " + ", ".join(f"{k}={v / 1e6:.2f}M" for k, v in allops.most_common(16)))

"""Per-source-line warp-stall samples and executed instructions from an ncu
report (cuda,sass source view): python tools/ncu_lines.py report kernel_regex [top]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(out.splitlines()))
fname = None
res = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] != "":
        def num(x):
            try:
                return int(float(x))
            except ValueError:
                return 0
        res.append((num(r[4]), num(r[7]), f"{fname}:{r[0]}", r[1].strip()[:80]))
tot = sum(x[0] for x in res)
print("total stall samples", tot)
for s, ie, loc, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{s:6d} {100 * s / max(tot, 1):5.1f}% {ie:9d}  {loc:22s} {src}")

"""Per-CUDA-source-line warp-stall samples and executed instructions from an
ncu report (source page, cuda,sass view).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


fname, hdr, recs = None, None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].isdigit():
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        st = sorted(((num(r[i]), h[6:]) for i, h in enumerate(hdr)
                     if h.startswith("stall_") and "Not Issued" not in h), reverse=True)[:2]
        recs.append((fname, int(r[0]), r[1].strip(), num(r[si]), num(r[ie]),
                     " ".join(f"{n}={v:.0f}" for v, n in st if v)))
tot = sum(x[3] for x in recs) or 1
itot = sum(x[4] for x in recs) or 1
print(f"samples {tot:.0f}  warp-instructions {itot:.0f}")
for f, ln, s, smp, ins, why in sorted(recs, key=lambda x: -x[3])[:top]:
    print(f"{f}:{ln:<5d} {100 * smp / tot:5.1f}% smp {100 * ins / itot:5.1f}% inst  {s[:60]:60s} {why}")

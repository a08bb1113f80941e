"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch
list: python tools/launch_summary.py launches.csv > summary.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows:
    name = re.sub(r"^void ", "", r[4])
    name = re.sub(r"\(.*$", "", name)
    tot[name] += float(r[14]) / 1e3
    cnt[name] += 1
s = sum(tot.values())
print("kernel,launches,total_us,share")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k},{cnt[k]},{tot[k]:.1f},{tot[k] / s:.3f}")

"""Condense ncu reports into profiles/ncu_summary.json (read by bench.py for
roofline.traffic): per library kernel kind, the DRAM bytes per launch and the
headline counters of the captured launches.
usage: python tools/ncu_to_json.py out.json report.ncu-rep [report2.ncu-rep ...]"""
import csv
import json
import subprocess
import sys

KIND = {"k_pass1": "ntt_pass1", "k_pass2": "ntt_pass2", "k_pass3": "ntt_pass3", "k_combine": "crt_combine",
        "k_quantize": "quantize", "k_tc_window": "direct", "k_outer_fwd": "other", "k_outer_inv": "other"}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}

out = {"source": sys.argv[2:], "kernels": {}}
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        base = name.split("(")[0].split("<")[0].split("::")[-1].strip().split()[-1]
        kind = KIND.get(base, base)
        rec = {"kernel": name[:120], "report": rep}
        for k in KEYS:
            if k in hdr:
                v, u = r[hdr.index(k)].replace(",", ""), units[hdr.index(k)]
                try:
                    rec[k] = float(v) * SCALE.get(u, 1)
                except ValueError:
                    rec[k] = v
        if "dram__bytes_read.sum" in rec:
            rec["dram_bytes_per_launch"] = rec["dram__bytes_read.sum"] + rec.get("dram__bytes_write.sum", 0)
        out["kernels"].setdefault(kind, rec)
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps({k: (v.get("dram_bytes_per_launch"), v.get("gpu__time_duration.sum")) for k, v in out["kernels"].items()}))

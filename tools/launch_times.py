"""Summarise an ncu launch list csv (gpu__time_duration.sum per launch):
usage: python tools/launch_times.py gpurun_out/x.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[i], rows[i + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in data:
    agg[r[ki].split("(")[0][:48]].append(float(r[vi].replace(",", "")))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} n={len(v):3d} mean_us={sum(v) / len(v) / 1e3:9.2f} last_us={v[-1] / 1e3:9.2f}")

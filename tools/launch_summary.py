"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel launches, total and mean duration, share of device time.

    python tools/launch_summary.py launches.csv [steps]
"""
import collections
import csv
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, data = None, []
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    k = d["Kernel Name"].split("(")[0][:64]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    per = f" {v[1] / steps / 1e3:8.2f}us/step" if steps else ""
    print(f"{k:64s} {v[0]:5d} {v[1] / 1e3:9.1f}us {v[1] / v[0] / 1e3:7.2f}us/launch "
          f"{100 * v[1] / tot:5.1f}%{per}")
print(f"total {tot / 1e3:.1f} us" + (f", {tot / steps / 1e3:.1f} us/step" if steps else ""))

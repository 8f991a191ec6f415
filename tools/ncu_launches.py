"""Summary of an ncu launch list (--metrics gpu__time_duration.sum --csv):
mean duration and share of the library's kernels per kernel name.
  python tools/ncu_launches.py launches.csv "title" > summary.txt"""
import collections
import csv
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
hdr, acc = None, collections.defaultdict(list)
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum" or not d["Kernel Name"].startswith("void k_"):
        continue
    acc[d["Kernel Name"]].append(float(d["Metric Value"].replace(",", "")) * UNIT[d["Metric Unit"]])
tot = sum(sum(v) for v in acc.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("(gpu__time_duration.sum, --clock-control none; cold-cache serialised launches: compare shares, not absolutes)")
for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    name = k.split("(")[0]
    print(f"{name:40s} launches {len(v):2d}  mean {sum(v) / len(v):8.1f} us  share of the fabf kernels {100 * sum(v) / tot:5.1f}%")

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
    agg.setdefault(d["Kernel Name"][:70], []).append(float(d["Metric Value"].replace(",", "")) * scale)
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{k:70s} n={len(v):3d} mean={sum(v) / len(v):9.1f} us  share={100 * sum(v) / tot:5.1f}%")

"""Per-kernel mean of each metric in an ncu --csv launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg.setdefault(d["Kernel Name"][:44], collections.defaultdict(list))[d["Metric Name"]].append(
            float(d["Metric Value"].replace(",", "")) if d["Metric Value"] not in ("n/a", "") else 0.0)
for k, v in agg.items():
    print(f"{k:44s} n={len(next(iter(v.values()))):3d}",
          " ".join(f"{m.split('.')[0].split('__')[1][:12]}={sum(x) / len(x):.4g}" for m, x in v.items()))

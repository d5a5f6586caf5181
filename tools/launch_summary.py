"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
agg = collections.OrderedDict()
for d in data:
    v = float(d["Metric Value"])
    unit = d["Metric Unit"]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
    name = d["Kernel Name"].split("(")[0][:70]
    key = (name, d.get("Grid Size", ""), d.get("Block Size", "")) if len(sys.argv) > 2 else name
    agg.setdefault(key, []).append(v * scale)
tot = sum(sum(v) for v in agg.values())
print(f"{len(data)} launches, total {tot / 1e3:.3f} ms")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:40]:
    print(f"{sum(v) / 1e3:10.3f} ms {100 * sum(v) / tot:5.1f}%  n={len(v):5d}  {k}")

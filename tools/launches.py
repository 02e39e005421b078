"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi = h.index("Kernel Name"), h.index("Metric Value")
ui = h.index("Metric Unit") if "Metric Unit" in h else None
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    name = r[ki].split("(")[0].split("::")[-1]
    v = float(r[mi].replace(",", "")) * scale.get(r[ui] if ui is not None else "ms", 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:32s} n={v[0]:5d} total={v[1]:9.3f} ms {100 * v[1] / tot:5.1f}%")
print(f"total {tot:.3f} ms")

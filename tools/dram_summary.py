"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv` log per kernel: launches, time, share, DRAM bytes per launch, achieved DRAM GB/s."""
import collections
import csv
import sys

SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mn, mv, mu, idi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
launch, names = collections.defaultdict(dict), {}
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    names[r[idi]] = r[ki].split("(")[0].split("::")[-1]
    launch[r[idi]][r[mn]] = float(r[mv].replace(",", "")) * SCALE.get(r[mu], 1.0)
agg = collections.OrderedDict()
for lid, m in launch.items():
    a = agg.setdefault(names[lid], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':32s} {'n':>4s} {'ms':>9s} {'share':>6s} {'read MB/l':>10s} {'write MB/l':>10s} {'DRAM GB/s':>9s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:32s} {v[0]:4d} {v[1] * 1e3:9.3f} {100 * v[1] / tot:5.1f}% {v[2] / v[0] / 1e6:10.1f} {v[3] / v[0] / 1e6:10.1f} "
          f"{(v[2] + v[3]) / v[1] / 1e9 if v[1] else 0.0:9.1f}")
print(f"total {tot * 1e3:.3f} ms")

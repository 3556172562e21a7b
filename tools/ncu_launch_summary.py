"""Aggregate an ncu --metrics gpu__time_duration.sum,dram__bytes_* launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    names[r[ii]] = r[ki]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    name = names[i].split("(")[0].replace("void ", "")
    a = agg[name]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>7s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:44]:44s} {a[0]:8d} {a[1] / 1e6:9.3f} {a[1] / tot:6.3f} {a[2] / a[0] / 1e6:10.1f} "
          f"{a[2] / a[1]:7.0f}")
print(f"total kernel time {tot / 1e6:.3f} ms (ncu: serialised, cold caches, clocks uncontrolled)")

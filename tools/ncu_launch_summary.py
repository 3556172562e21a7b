"""Aggregate an ncu --metrics gpu__time_duration.sum,dram__bytes_* launch list per kernel.

MB/launch averages over every launch; MB/active averages over launches that
moved more than 1 MB (the step kernels of a cycle that already stopped
early-exit and move nothing)."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
ui = h.index("Metric Unit") if "Metric Unit" in h else None
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
         "msecond": 1e6}
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    v = float(r[vi].replace(",", ""))
    if ui is not None:
        v *= scale.get(r[ui], 1)
    per[r[ii]][r[mi]] = v
    names[r[ii]] = r[ki]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0, 0.0, 0.0])
for i, m in per.items():
    name = names[i].split("(")[0].replace("void ", "")
    a = agg[name]
    t = m.get("gpu__time_duration.sum", 0.0)
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a[0] += 1
    a[1] += t
    a[2] += b
    if b > 1e6:
        a[3] += 1
        a[4] += t
        a[5] += b
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'MB/launch':>10s} "
      f"{'active':>6s} {'MB/active':>10s} {'GB/s':>7s}")
out = {}
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    act = a[5] / a[3] / 1e6 if a[3] else 0.0
    gbs = a[5] / a[4] if a[4] else 0.0
    print(f"{k[:44]:44s} {a[0]:8d} {a[1] / 1e6:9.3f} {a[1] / tot:6.3f} {a[2] / a[0] / 1e6:10.1f} "
          f"{a[3]:6d} {act:10.1f} {gbs:7.0f}")
    out[k] = {"launches": a[0], "active_launches": a[3], "ms": a[1] / 1e6,
              "dram_bytes_per_active_launch": int(a[5] / a[3]) if a[3] else 0}
print(f"total kernel time {tot / 1e6:.3f} ms (ncu: serialised, cold caches, clocks uncontrolled)")
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)

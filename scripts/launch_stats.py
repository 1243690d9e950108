"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
metric = "gpu__time_duration.sum"
data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr_i + 1:] if len(r) > vi and r[mi] == metric]
by = collections.defaultdict(dict)
for r in rows[hdr_i + 1:]:
    if len(r) > vi:
        by[r[hdr.index("ID")]][r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in data:
    m = re.search(r"(\w+_kernel)", k)
    name = m.group(1) if m else k[:40]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{len(data)} launches, {tot/1e3:.1f} us total")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:30s} {c:5d} {v/1e3:10.1f} us {100*v/tot:5.1f}%  avg {v/c/1e3:8.2f} us")
names = {}
for r in rows[hdr_i + 1:]:
    if len(r) > vi:
        m = re.search(r"(\w+_kernel)", r[ki])
        names[r[hdr.index("ID")]] = m.group(1) if m else r[ki][:40]
traffic = collections.defaultdict(lambda: [0, 0.0])
for i, v in by.items():
    if "dram__bytes_read.sum" in v:
        unit_scale = 1.0
        traffic[names[i]][0] += 1
        traffic[names[i]][1] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
if traffic:
    print("DRAM traffic per launch (read + write, as ncu reports the unit):")
    for k, (c, v) in sorted(traffic.items(), key=lambda x: -x[1][1]):
        print(f"  {k:30s} {c:5d} launches  avg {v / c:12.1f}")
for name in sys.argv[2:]:
    seq = [v for k, v in data if name in k]
    print(name, [round(x / 1e3, 1) for x in seq[-48:]])

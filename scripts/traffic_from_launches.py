"""Average DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per
launch of each kernel in an ncu launch list (one solve, --clock-control
none) -> profiles/traffic.json, read by bench.py for roofline.traffic."""
import collections
import csv
import json
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = collections.defaultdict(dict)
name = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    m = re.search(r"(\w+_kernel)", r[ki])
    name[r[ii]] = m.group(1) if m else r[ki][:40]
    if r[mi].startswith("dram__bytes"):
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
agg = collections.defaultdict(lambda: [0, 0.0])
for i, v in per.items():
    agg[name[i]][0] += 1
    agg[name[i]][1] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
out = {k: {"launches": c, "bytes_per_launch": round(b / c)} for k, (c, b) in agg.items()}
out["_source"] = src
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))

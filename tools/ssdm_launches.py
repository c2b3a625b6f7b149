"""Summarise an ncu --csv launch list (one row per metric) by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
for n, (c, us, mb) in agg.items():
    print(f"{n:42s} x{c:3d}  {us / c:9.1f} us/launch  {mb / c:9.1f} MB/launch  "
          f"{mb / us if us else 0:6.2f} TB/s")

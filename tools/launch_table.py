"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel name, launches,
total and mean time. usage: python tools/launch_table.py launches.csv [divide_by]"""
import csv
import re
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
head = rows[h]
ki, vi = head.index("Kernel Name"), head.index("Metric Value")
agg = OrderedDict()
seq = []
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    n = re.sub(r"\(.*", "", r[ki].replace("(anonymous namespace)::", "").replace("sfb::", "").replace("void ", ""))
    n = re.sub(r"<unnamed>::", "", n)
    v = float(r[vi].replace(",", ""))
    a = agg.setdefault(n, [0.0, 0])
    a[0] += v
    a[1] += 1
    seq.append((n, v))
tot = sum(a[0] for a in agg.values())
for n, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n[:70]:70s} {c:5d} {v / 1e6 / div:9.3f} ms  {100 * v / tot:5.1f}%")
if "-seq" in sys.argv:
    for n, v in seq:
        print(f"  {n[:70]:70s} {v / 1e3:9.1f} us")

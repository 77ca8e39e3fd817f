"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import re
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    name = re.sub(r"plnmf::|<unnamed>::|\(anonymous namespace\)::", "", name)[:70]
    tot.setdefault(name, []).append(float(r[vi].replace(",", "")))
grand = sum(sum(v) for v in tot.values())
for n, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
    print(f"{n:70s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f}us total={sum(v) / 1e3:9.1f}us {100 * sum(v) / grand:5.1f}%")

"""Hot SASS lines of a `ncu --page source --csv` export: stall samples by opcode and the top lines.
   python tools/ncu_hot.py gpurun_out/one_source.csv [n]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[wi]), float(r[ei]), r[0][-5:], r[si].strip()[:100]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1.0
print("samples", tot, "instructions", sum(d[1] for d in data))
op, opi = Counter(), Counter()
for s, i, a, src in data:
    o = src.split()[1] if src.startswith("@") else (src.split()[0] if src else "?")
    op[o.split(".")[0]] += s
    opi[o.split(".")[0]] += i
for o, v in op.most_common(10):
    print(f"{o:10s} stall {100 * v / tot:5.1f}%  instr {opi[o]:.3g}")
for s, i, a, src in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{100 * s / tot:5.1f}% {i:11.0f} {a} {src}")

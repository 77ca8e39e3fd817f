"""Top SASS lines of a `ncu --page source --csv` export with their dominant stall reasons.
   python tools/ncu_stalls.py gpurun_out/one_source.csv [n] [addr_lo addr_hi]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
st = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lo, hi = (int(sys.argv[3], 16), int(sys.argv[4], 16)) if len(sys.argv) > 4 else (0, 1 << 62)
data = []
for r in rows[2:]:
    try:
        a = int(r[0][-5:], 16)
        if lo <= a < hi:
            data.append((float(r[wi]), float(r[ei]), r[0][-5:], r[si].strip()[:60], r))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1.0
reasons = {}
for d in data:
    for i, c in st:
        try:
            reasons[c] = reasons.get(c, 0) + float(d[4][i])
        except ValueError:
            pass
print("samples", tot, " by reason:", ", ".join(f"{c[6:]} {100 * v / tot:.1f}%" for c, v in sorted(reasons.items(), key=lambda x: -x[1])[:8]))
for s, i, a, src, r in sorted(data, key=lambda x: -x[0])[:n]:
    top = sorted(((float(r[j]) if r[j] else 0.0, c[6:]) for j, c in st), reverse=True)[:2]
    print(f"{100 * s / tot:5.1f}% {i:9.0f} {a} {src:60s} " + " ".join(f"{c}:{v:.0f}" for v, c in top if v))

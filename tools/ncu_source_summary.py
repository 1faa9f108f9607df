"""Summarise an ncu --page source --csv export: stall reasons and hottest SASS."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[si] or 0) for r in data)
agg = collections.Counter()
for r in data:
    for c in reasons:
        agg[c] += float(r[h.index(c)] or 0)
print(f"total stall samples {tot:.0f}")
for c, v in agg.most_common(10):
    print(f"  {c:28s} {100 * v / max(tot, 1):5.1f}%")
op = collections.Counter()
for r in data:
    opc = r[1].strip().split()[0] if r[1].strip() else "?"
    if opc.startswith("@"):
        opc = r[1].strip().split()[1]
    op[opc.split(".")[0]] += float(r[si] or 0)
print("by opcode:", ", ".join(f"{k} {100 * v / max(tot, 1):.1f}%" for k, v in op.most_common(12)))
print("hottest instructions:")
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:top]:
    det = {c.replace("stall_", ""): float(r[h.index(c)] or 0) for c in reasons}
    best = sorted(det.items(), key=lambda x: -x[1])[:3]
    print(f"  {float(r[si]):6.0f} {r[0][-5:]} {r[1].strip()[:60]:60s} {best}")

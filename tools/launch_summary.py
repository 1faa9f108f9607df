"""Per-kernel summary of an ncu launch list (ncu --metrics gpu__time_duration.sum --csv --log-file F):
python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches_summary.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1], errors="replace")) if len(r) > 5]
hd = next(r for r in rows if "Kernel Name" in r)
ik, iv, iu = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Metric Unit")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if r is hd or len(r) <= iv or r[ik] == "Kernel Name":
        continue
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r[iu].strip(), 1e-6)
    tot[r[ik]] += v * scale
    cnt[r[ik]] += 1
allms = sum(tot.values()) or 1.0
print("launches  total_ms  share  kernel")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{cnt[k]:8d} {v:9.3f} {100 * v / allms:5.1f}%  {k[:110]}")

"""Summaries of one round's ncu captures (gpurun_out/) for profiles/:
launch list (launches.csv) -> per-kernel totals; prof_sweep.ncu-rep -> key counters + stall
reasons + hottest SASS of the persistent HALS sweep; prof_i8.ncu-rep -> per-launch table of the
INT8 digit GEMMs.  Usage: python tools/ncu_summaries.py <gpurun_out dir> <out prefix>"""
import collections
import csv
import io
import os
import subprocess
import sys

src, pre = sys.argv[1], sys.argv[2]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


# 1. launch list
rows = list(csv.reader(open(os.path.join(src, "launches.csv"))))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hd = rows[h]
ki, mi, vi = hd.index("Kernel Name"), hd.index("Metric Name"), hd.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[h + 1:]:
    if len(r) == len(hd) and r[mi] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", ""))
        unit = r[hd.index("Metric Unit")]
        ms = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e3) * v
        tot[r[ki]] += ms
        cnt[r[ki]] += 1
all_ms = sum(tot.values())
with open(pre + "_launches_summary.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 2 --warmup 3 "
            "--no-e2e --no-cpu\n# (serialised, cold-cache launch times; includes torch's data generation, the "
            "one-time X digit cuts and the TF32\n#  variant's run)\nlaunches  total_ms  share  kernel\n")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write(f"{cnt[k]:8d} {v:9.3f} {100 * v / all_ms:5.1f}%  {k[:100]}\n")

# 2. sweep capture
rep = os.path.join(src, "prof_sweep.ncu-rep")
raw = ncu_csv(["-i", rep, "--page", "raw"])
hd, units, vals = raw[0], raw[1], raw[2]
want = ["Block Size", "Grid Size", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
with open(pre + "_sweep_ncu.txt", "w") as f:
    f.write("# ncu --set full --clock-control none, one launch of hals::sweep_ws<128,0,0,1> (persistent: all sweeps "
            "of one inner solve)\n# python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu, -k regex:sweep_ws -s 2 -c 1\n")
    for w in want:
        if w in hd:
            i = hd.index(w)
            f.write(f"{w} = {vals[i]} {units[i]}\n")
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_source_summary.py"), rep, "12"],
                         capture_output=True, text=True).stdout
    f.write(out)

# 3. int8 digit GEMMs
raw = ncu_csv(["-i", os.path.join(src, "prof_i8.ncu-rep"), "--page", "raw"])
hd, units = raw[0], raw[1]
cols = ["Kernel Name", "Grid Size", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
idx = [hd.index(c) for c in cols if c in hd]
with open(pre + "_int8_gemm_ncu.txt", "w") as f:
    f.write("# ncu --set full --clock-control none of int8 digit GEMM launches (cuBLASLt), python bench.py --steps 2 "
            "--warmup 3\n# columns: " + ", ".join(f"{hd[i]} [{units[i]}]" for i in idx) + "\n")
    for r in raw[2:]:
        f.write("  ".join(r[i][:60] for i in idx) + "\n")
print("wrote", pre + "_launches_summary.txt", pre + "_sweep_ncu.txt", pre + "_int8_gemm_ncu.txt")

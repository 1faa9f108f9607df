"""One-page summary of an ncu --set full capture (key counters, stall reasons, hottest SASS) for
profiles/.  Usage: python tools/ncu_report.py <capture.ncu-rep> <title> [> profiles/rNN_x_ncu.txt]"""
import csv
import io
import os
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(out)))
hd, units, vals = raw[0], raw[1], raw[2]
want = ["Kernel Name", "Block Size", "Grid Size", "gpu__time_duration.sum", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
        "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
print(f"# {title}")
print(f"# ncu --set full --clock-control none --import-source on ({os.path.basename(rep)}); "
      "cold-cache, serialised launch")
for w in want:
    if w in hd:
        i = hd.index(w)
        print(f"{w.split('TriageCompute.')[-1]} = {vals[i][:110]} {units[i]}")
stalls = [(float(vals[i].replace(",", "") or 0), hd[i]) for i in range(len(hd))
          if hd[i].startswith("smsp__average_warp_latency_issue_stalled_") is False
          and hd[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not hd[i].endswith("not_issued")
          and vals[i].replace(",", "").replace(".", "").isdigit()]
tot = sum(v for v, _ in stalls) or 1.0
print("## warp-state samples (pc sampling), top 8")
for v, n in sorted(stalls, reverse=True)[:8]:
    print(f"  {100 * v / tot:5.1f}%  {n.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
src = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_source_summary.py"), rep, "10"],
                     capture_output=True, text=True).stdout
print(src)

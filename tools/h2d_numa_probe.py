"""Pinned host->device bandwidth of an 8.6 GB buffer with the process left where the scheduler
put it vs bound to the GPU's NVML CPU affinity (the GPU-local NUMA node) before allocating."""
import os, sys, time
import torch
import pynvml

def bw(tag):
    n = 32768 * 32768
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{tag}: {n * 8 / dt / 1e9:.1f} GB/s (affinity {sorted(os.sched_getaffinity(0))[:4]}... {len(os.sched_getaffinity(0))} cpus)")
    del h, d
    torch.cuda.empty_cache()

torch.cuda.init()
bw("default")
pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
words = pynvml.nvmlDeviceGetCpuAffinity(hnd, (os.cpu_count() + 63) // 64)
cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
print("GPU0 local cpus:", len(cpus), "of", os.cpu_count())
os.sched_setaffinity(0, cpus)
bw("bound to the GPU's cpus")

"""Per-sweep cost of the persistent sweep kernel vs the number of sweeps in one solve: run under ncu
(tools/gpu_sweep_scan.sh), whose launch durations are the device times.  C5 shape, forced sweep
counts (stall fraction 1e-300)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1805_06604_b200 as E

r, n = 128, 32768
rng = np.random.default_rng(0)
w = rng.random((4096, r))
G = w.T @ w
C = G @ rng.random((r, n)) * 0.9
h0 = rng.random((r, n))
ctx = E.Context()
if os.environ.get("SWEEP_PREC") == "tf32":   # the TF32 variant's sweep kernels (hals_rl.cuh / sweep_tf32.cuh)
    ctx.set_precision(E.Precision.tf32)
for ms in (2, 4, 8, 16, 32, 64, 129, 129, 64, 8):
    t = time.perf_counter()
    h, sw = ctx.hals_solve(G, C, h0, ms, 1e-300)
    dt = time.perf_counter() - t
    print(f"max_sweeps={ms:4d} sweeps={sw:4d} wall={dt*1e3:8.2f} ms", flush=True)

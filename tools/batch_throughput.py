"""C1-class runs per second: the packed backend (one launch, one CTA per run) vs run_batch on
streams, e-ahals-hp3, 200 outer iterations per run (config 1's protocol)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1805_06604_b200 as E
from paper_1805_06604_b200 import data as Dt

B = int(os.environ.get("BATCH", "1184"))
x = Dt.gen_lowrank(200, 200, 20, 1)
probs = [(x, *Dt.random_init(200, 200, 20, 100 + s)) for s in range(B)]
cfg = E.algorithm_config("e-ahals-hp3")
cfg.max_outer_iterations = 200
E.run_batch_packed(probs[:16], cfg)                        # warm-up
# device time of the batch kernel alone (CUDA events around the C-ABI call's launch are not
# reachable from here: time the C call with records off, and with records on)
import ctypes as C
from paper_1805_06604_b200 import _lib as L
xs = np.ascontiguousarray(np.stack([p[0] for p in probs])); ws = np.ascontiguousarray(np.stack([p[1] for p in probs]))
hs = np.ascontiguousarray(np.stack([p[2] for p in probs]))
c = cfg.to_c(E.TimingMode.none)
nit = np.zeros(B, dtype=np.int32); st = np.zeros(B, dtype=np.int32)
wo = np.empty((B, 200, 20)); ho = np.empty((B, 20, 200)); nx = np.empty(B)
ip = C.POINTER(C.c_int32)
ctx = E.default_context()
lib = L.load()
for rep in range(2):
    t = time.perf_counter()
    rc = lib.enmf_gpu_run_batch_dense(ctx._h, B, xs.ctypes.data, 200, 200, ws.ctypes.data, hs.ctypes.data, 20, C.byref(c),
                                      None, 0, nit.ctypes.data_as(ip), st.ctypes.data_as(ip), wo.ctypes.data,
                                      ho.ctypes.data, nx.ctypes.data)
    dt = time.perf_counter() - t
print(f"C-ABI call without records (upload + kernel + download): {dt:.3f} s = {B / dt:.0f} runs/s, rc {rc}")
best = 1e9
for rep in range(3):
    t = time.perf_counter()
    out = E.run_batch_packed(probs, cfg)
    best = min(best, time.perf_counter() - t)
print(f"packed: {B} runs x 200 iterations in {best:.3f} s = {B / best:.0f} runs/s "
      f"(final rel. error of run 0: {out[0].final_relative_error():.6e})")
for alg in ("e-anls-hp1", "ahals"):
    ca = E.algorithm_config(alg)
    ca.max_outer_iterations = 200
    E.run_batch_packed(probs[:16], ca)
    t = time.perf_counter()
    E.run_batch_packed(probs, ca)
    dt = time.perf_counter() - t
    print(f"packed {alg}: {B} runs in {dt:.3f} s = {B / dt:.0f} runs/s (through Python)")
nb = min(B, 64)
t = time.perf_counter()
E.run_batch(probs[:nb], cfg, backend="streams", streams=16)
dt = time.perf_counter() - t
print(f"streams: {nb} runs in {dt:.3f} s = {nb / dt:.0f} runs/s")

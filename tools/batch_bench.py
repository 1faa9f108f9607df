"""Throughput of many small runs (BASELINE configs[0] shape: 200×200 r=20, E-A-HALS hp3,
200 iterations — the paper's 10 datasets × 10 inits protocol) on one B200: one run at a
time vs run_batch with several contexts/streams in flight."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_06604_b200 as E

R = int(os.environ.get("RUNS", "100"))
rng = np.random.default_rng(0)
probs = []
for i in range(R):
    x = rng.random((200, 20)) @ rng.random((20, 200))
    probs.append((x, rng.random((200, 20)), rng.random((20, 200))))
cfg = E.algorithm_config("e-ahals-hp3")
cfg.max_outer_iterations = 200
ctx = E.Context()
ctx.run(*probs[0], cfg, E.TimingMode.none)            # warm-up
t = time.perf_counter()
for p in probs:
    ctx.run(*p, cfg, E.TimingMode.none)
seq = time.perf_counter() - t
print(f"sequential: {R} runs in {seq:.3f} s = {R / seq:.1f} runs/s")
for k in (8, 16, 32, 64):
    E.run_batch(probs[:k], cfg, streams=k)           # warm-up
    t = time.perf_counter()
    E.run_batch(probs, cfg, streams=k)
    dt = time.perf_counter() - t
    print(f"run_batch streams={k}: {R} runs in {dt:.3f} s = {R / dt:.1f} runs/s ({seq / dt:.1f}x)")

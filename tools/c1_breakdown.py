"""Where a single small run's time goes (C1 shape): load, begin (graph capture), K iterations, end."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_06604_b200 as E
rng = np.random.default_rng(0)
x = rng.random((200, 20)) @ rng.random((20, 200)); w0 = rng.random((200, 20)); h0 = rng.random((20, 200))
cfg = E.algorithm_config("e-ahals-hp3"); cfg.max_outer_iterations = 200
ctx = E.Context()
for rep in range(3):
    t0 = time.perf_counter(); ctx.load(x)
    t1 = time.perf_counter(); ctx.begin(w0, h0, cfg)
    t2 = time.perf_counter(); ctx.step(200)
    t3 = time.perf_counter(); recs = ctx.sync()
    t4 = time.perf_counter(); w = np.empty((200, 20)); h = np.empty((20, 200)); ctx.end(w.ctypes.data, h.ctypes.data)
    t5 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} ms  begin {1e3*(t2-t1):.2f}  step-enqueue {1e3*(t3-t2):.2f}  sync {1e3*(t4-t3):.2f}  end {1e3*(t5-t4):.2f}"
          f"  sweeps/iter {np.mean([r.inner_h_count + r.inner_w_count for r in recs[1:]]):.1f}")
print("kernels per run:", ctx.kernel_launches)

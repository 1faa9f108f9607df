"""Times one HALS sweep kernel variant at C5 size through enmf_gpu_hals_solve
(ENMF_HALS_KERNEL selects the variant).  Prints µs per sweep."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_06604_b200 as E

LONG = int(os.environ.get("SWEEP_LONG", "40"))
r, n = int(os.environ.get("SWEEP_R", "128")), int(os.environ.get("SWEEP_N", "32768"))
rng = np.random.default_rng(0)
w = rng.random((4096, r))
G = w.T @ w
C = G @ rng.random((r, n)) * 0.9
h0 = rng.random((r, n))
ctx = E.Context()
ctx.hals_solve(G, C, h0, 8, 1e-12)          # warm-up
best = {}
for rep in range(3):
    for ms in (8, LONG):
        t = time.perf_counter()
        h, sw = ctx.hals_solve(G, C, h0, ms, 1e-12)
        dt = time.perf_counter() - t
        best[ms] = min(best.get(ms, 1e9), dt)
        print(f"{os.environ.get('ENMF_HALS_KERNEL', 'default')}: max_sweeps={ms} sweeps={sw} total={dt*1e3:.2f} ms")
print(f"{os.environ.get('ENMF_HALS_KERNEL', 'default')}: {(best[LONG] - best[8]) / (LONG - 8) * 1e6:.1f} us per sweep (best-of-3 difference)")

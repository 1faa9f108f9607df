"""Per-phase device times of one outer iteration (enmf_gpu_step_profiled) on the BASELINE C2 /
C3 / C4 shapes (python tools/small_phases.py c2|c3|c4): where a latency-bound iteration goes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_06604_b200 as E
import bench

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctx = E.Context(0)
if which == "c4":
    m, n, r, alg = 30000, 10000, 20, "e-ahals-hp3"
    off, cidx, vals = bench.gen_docs_csr(m, n, 404)
    ctx.load_csr(off, cidx, vals, m, n)
    rng = np.random.default_rng(405)
else:
    x, r, alg, iters = bench.gen_dense_config(which, 505)
    m, n = x.shape
    ctx.load(x)
    rng = np.random.default_rng(506)
w0, h0 = rng.random((m, r)), rng.random((r, n))
cfg = E.algorithm_config(alg)
cfg.max_outer_iterations = 60
ctx.begin(w0, h0, cfg)
ctx.step(40)
ctx.sync()
for _ in range(3):
    ph = ctx.step_profiled()
    print(which, " ".join(f"{k}={v:.4f}" for k, v in ph.items()))
ctx.sync()
ctx.end()
ctx.close()

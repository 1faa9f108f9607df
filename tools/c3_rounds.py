import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1805_06604_b200 as E
import bench
x, r, alg, iters = bench.gen_dense_config("c3", 505)
m, n = x.shape
rng = np.random.default_rng(506)
w0, h0 = rng.random((m, r)), rng.random((r, n))
cfg = E.algorithm_config(alg); cfg.max_outer_iterations = 30
ctx = E.Context(0)
rec = ctx.run(x, w0, h0, cfg, E.TimingMode.none)
print("h rounds", rec.column("inner_h_count")[:30])
print("w rounds", rec.column("inner_w_count")[:30])

import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1805_06604_b200 as E
from oracle.oracle import Oracle, preset
port = Oracle("port")
m, n, r = 37, 301, 1
rng = np.random.default_rng(m + n + r)
x = rng.random((m, r)) @ rng.random((r, n)) + np.abs(0.01 * rng.standard_normal((m, n)))
w0, h0 = port.random_init(m, n, r, 3)
c = E.algorithm_config("e-ahals-hp3"); c.max_outer_iterations = 8
rec = E.run_batch_packed([(x, w0, h0)], c)[0]
ref = port.run_dense(x, w0, h0, preset("e-ahals-hp3", max_outer_iterations=8))
one = E.Context().run(x, w0, h0, c, E.TimingMode.none)
print("err packed", rec.column("error")); print("err oracle", ref[0]["error"]); print("err engine", one.column("error"))
print("rs", rec.column("restarted").astype(int), ref[0]["restarted"], one.column("restarted").astype(int))
print("ih", rec.column("inner_h_count"), ref[0]["inner_h"], one.column("inner_h_count"))
print("iw", rec.column("inner_w_count"), ref[0]["inner_w"], one.column("inner_w_count"))

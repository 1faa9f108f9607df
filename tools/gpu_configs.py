"""Times the BASELINE parity configs C1-C3 end to end through the C-ABI and
checks them against the oracle (short runs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_06604_b200 as E
from oracle.oracle import Oracle, preset

P = Oracle("port")
ctx = E.Context()
cases = [("C1 e-ahals-hp3 200x200 r20", lambda: P.gen_lowrank(200, 200, 20, 1), 200, 200, 20, "e-ahals-hp3", 200, 200),
         ("C2 e-ahals-hp3 10304x400 r40", lambda: P.gen_config(2, 10304, 400, 40, 1), 10304, 400, 40, "e-ahals-hp3", 500, 10),
         ("C3 e-anls-hp1 2000x2000 r30", lambda: P.gen_config(3, 2000, 2000, 30, 1), 2000, 2000, 30, "e-anls-hp1", 100, 3)]
for name, gen, m, n, r, alg, iters, ref_iters in cases:
    x = gen()
    w0, h0 = P.random_init(m, n, r, 2)
    cfg = E.algorithm_config(alg)
    cfg.max_outer_iterations = iters
    ctx.run(x, w0, h0, cfg, E.TimingMode.none)     # warm-up (graph build, allocations)
    t = time.perf_counter()
    rec = ctx.run(x, w0, h0, cfg, E.TimingMode.none)
    dt = time.perf_counter() - t
    t = time.perf_counter()
    ref = P.run_dense(x, w0, h0, preset(alg, max_outer_iterations=ref_iters))
    dtc = time.perf_counter() - t
    e = rec.column("error")[: ref_iters + 1]
    dev = np.max(np.abs(e - ref[0]["error"]) / ref[0]["error"])
    same = np.array_equal(rec.column("restarted")[: ref_iters + 1].astype(np.int32), ref[0]["restarted"])
    print(f"{name}: GPU {iters} it in {dt*1e3:.1f} ms ({iters/dt:.1f} it/s, e2e incl. copies); "
          f"oracle {ref_iters} it {dtc:.2f} s ({ref_iters/dtc:.2f} it/s); first {ref_iters} it: restarts equal {same}, "
          f"max rel err dev {dev:.2e}; final rel {rec.final_relative_error():.6e}; "
          f"sweeps/rounds H {np.mean(rec.column('inner_h_count')[1:]):.1f} W {np.mean(rec.column('inner_w_count')[1:]):.1f}")

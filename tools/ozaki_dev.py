"""Deviation of the INT8-digit product path from the oracle (the parity test's C5-like 4096²
r=64 case and the wide-dynamic-range case), printed rather than asserted: for A/B of digit
schemes (ENMF_GPU_LIB selects a build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_06604_b200 as E
from oracle.oracle import Oracle, preset

port = Oracle("port")
ctx = E.Context(0)
for name, wide, r, it in (("c5like", False, 64, 6), ("wide", True, 32, 5)):
    m = n = 4096
    rng = np.random.default_rng(21 if not wide else 41)
    x = rng.random((m, r)) @ rng.random((r, n)) + np.abs(0.01 * rng.standard_normal((m, n)))
    if wide:
        x *= 10.0 ** rng.uniform(-3, 3, (m, 1))
        x *= 10.0 ** rng.uniform(-3, 3, (1, n))
    w0, h0 = port.random_init(m, n, r, 22 if not wide else 42)
    cfg = E.algorithm_config("e-ahals-hp3")
    cfg.max_outer_iterations = it
    ref, wr, hr, _ = port.run_dense(x, w0, h0, preset("e-ahals-hp3", max_outer_iterations=it))
    rec = ctx.run(x, w0, h0, cfg, E.TimingMode.none)
    err = rec.column("error")
    dev = np.abs(err - ref["error"]) / ref["error"]
    fw = np.max(np.abs(rec.factors.w - wr)) / np.max(np.abs(wr))
    fh = np.max(np.abs(rec.factors.h - hr)) / np.max(np.abs(hr))
    same = np.array_equal(rec.column("restarted").astype(np.int32), ref["restarted"]) and \
        np.array_equal(rec.column("inner_h_count"), ref["inner_h"]) and np.array_equal(rec.column("inner_w_count"), ref["inner_w"])
    print(f"{os.environ.get('ENMF_GPU_LIB', 'in-tree')} {name}: max rel dev of e {dev.max():.3e} "
          f"(per iteration {' '.join(f'{d:.1e}' for d in dev)}), W {fw:.2e}, H {fh:.2e}, decisions identical {same}")

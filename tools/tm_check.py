"""sweep_tm vs sweep_ws (ENMF_HALS_KERNEL=wsp) on the kernel-level hals_solve at r = 128: prints the
sweep count and a checksum of H per tiles-per-sub-partition case (run once per kernel variant)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1805_06604_b200 as E

ctx = E.Context(0)
for nt in [int(v) for v in (sys.argv[1:] or ["1", "4", "6", "7", "8"])]:
    r, n = 128, 148 * 4 * 8 * nt
    rng = np.random.default_rng(nt)
    w = rng.random((300, r))
    g = w.T @ w
    x = rng.random((300, n))
    c = w.T @ x
    h0 = rng.random((r, n))
    h, s = ctx.hals_solve(g, c, h0, 200, 0.01)
    print(f"nt {nt}: sweeps {s} sum {h.sum():.15e} max {h.max():.6e}", flush=True)

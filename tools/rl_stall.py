import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1805_06604_b200 as E
ctx = E.Context(0)
for (r, n, ms, stall) in [(128, 29600, 40, 0.01), (100, 5000, 40, 0.01), (72, 777, 40, 0.3), (128, 32768, 129, 0.001), (40, 3000, 3, 1e-300), (128, 5000, 1, 0.01)]:
    rng = np.random.default_rng(r + n)
    w = rng.random((600, r)); g = w.T @ w; c = w.T @ rng.random((600, n)); h0 = rng.random((r, n))
    ctx.set_precision(E.Precision.fp64); h64, s64 = ctx.hals_solve(g, c, h0, ms, stall)
    ctx.set_precision(E.Precision.tf32); h32, s32 = ctx.hals_solve(g, c, h0, ms, stall)
    h32b, s32b = ctx.hals_solve(g, c, h0, ms, stall)
    f = lambda h: 0.5 * np.sum(h * (g @ h)) - np.sum(c * h)
    print(f"r {r} n {n} cap {ms} stall {stall}: sweeps fp64 {s64} tf32 {s32}/{s32b} repeat-identical {np.array_equal(h32, h32b)} obj fp64 {f(h64):.8e} tf32 {f(h32):.8e} min {h32.min():.1e}", flush=True)

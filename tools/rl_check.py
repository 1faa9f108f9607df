"""TF32 right-looking sweep (hals_rl.cuh; ENMF_TF32_SWEEP=mma: the mma.sync kernel) vs the FP64
sweep on the kernel-level hals_solve: deviation of H after 1, 4, 16, 64 forced sweeps."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1805_06604_b200 as E

ctx = E.Context(0)
for (r, n) in [(128, 148 * 200), (100, 5000)]:
    rng = np.random.default_rng(r + n)
    w = rng.random((600, r))
    g = w.T @ w
    x = rng.random((600, n))
    c = w.T @ x
    h0 = rng.random((r, n))
    for ms in (1, 4, 16, 64):
        ctx.set_precision(E.Precision.fp64)
        h64, s64 = ctx.hals_solve(g, c, h0, ms, 1e-300)
        ctx.set_precision(E.Precision.tf32)
        h32, s32 = ctx.hals_solve(g, c, h0, ms, 1e-300)
        res64 = np.linalg.norm(c - g @ h64 * (h64 > 0))
        d = np.abs(h32 - h64)
        print(f"r {r} n {n} sweeps {s64}/{s32}: max dev {d.max() / h64.max():.3e} mean dev {d.mean() / h64.mean():.3e}; "
              f"objective fp64 {0.5 * np.sum(h64 * (g @ h64)) - np.sum(c * h64):.9e} tf32 {0.5 * np.sum(h32 * (g @ h32)) - np.sum(c * h32):.9e}",
              flush=True)

"""TF32 variant at small ranks: iterations/s with the tcgen05 right-looking sweeps (default) and with
the mma.sync kernel (ENMF_TF32_SWEEP=mma) — run once per mode."""
import sys, time, os
import numpy as np
sys.path.insert(0, ".")
import paper_1805_06604_b200 as E
ctx = E.Context(0)
for (m, n, r, it) in [(10304, 400, 40, 300), (200, 200, 20, 200), (2000, 2000, 30, 100), (6000, 5000, 64, 60)]:
    rng = np.random.default_rng(m + n)
    x = rng.random((m, r)) @ rng.random((r, n)) + np.abs(0.01 * rng.standard_normal((m, n)))
    w0, h0 = rng.random((m, r)), rng.random((r, n))
    c = E.algorithm_config("e-ahals-hp3"); c.max_outer_iterations = it; c.precision = E.Precision.tf32
    ctx.load(x)
    best = 1e9
    for rep in range(3):
        t = time.perf_counter(); rec = ctx._solve_host(w0, h0, m, n, c, E.TimingMode.none); best = min(best, time.perf_counter() - t)
    print(f"{os.environ.get('ENMF_TF32_SWEEP','rl')}: {m}x{n} r={r}: {it / best:.0f} it/s, final rel err {rec.final_relative_error():.6e}, sweeps h/w {rec.column('inner_h_count')[1:].mean():.1f}/{rec.column('inner_w_count')[1:].mean():.1f}", flush=True)

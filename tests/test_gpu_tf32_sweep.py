"""GPU tier: the TF32 variant's HALS sweeps at kernel level (enmf_gpu_hals_solve in TF32 precision)
against the FP64 sweeps of the same problem — the tcgen05 right-looking kernel (hals_rl.cuh:
residual in tensor memory, rank-8 kind::tf32 updates) for r <= 128 with 256 <= N and every CTA's
columns resident, the mma.sync kernel (sweep_tf32.cuh) otherwise.  TF32 is a reduced-precision variant
(north_star: final relative error within 1e-4), so the check is on the NNLS objective
f(H) = ½⟨H, G·H⟩ − ⟨C, H⟩ the sweeps minimise (nnls.hpp:111-176), not on H entry by entry."""
import numpy as np
import pytest

import paper_1805_06604_b200 as E

pytestmark = pytest.mark.gpu


def _objective(g, c, h):
    return 0.5 * np.sum(h * (g @ h)) - np.sum(c * h)


@pytest.mark.parametrize("r,n,sweeps", [
    (128, 5000, 30),     # 34 columns per CTA: tile 0 only
    (128, 29600, 12),    # 200 columns per CTA: both tiles
    (100, 300, 30),      # ragged r, few CTAs
    (72, 777, 30),       # ragged r and N
    (128, 40000, 6),     # more than 256 columns per CTA: falls back to the mma.sync kernel
    (64, 900, 20),       # 8 row blocks of 16
    (20, 3000, 20),      # 3 row blocks
    (40, 200, 20),       # fewer than 256 columns: mma.sync kernel
])
def test_tf32_sweeps_reach_the_fp64_objective(r, n, sweeps):
    ctx = E.Context(0)
    rng = np.random.default_rng(r * 1000 + n)
    w = rng.random((400, r))
    g = w.T @ w
    c = w.T @ rng.random((400, n))
    h0 = rng.random((r, n))
    f0 = _objective(g, c, h0)
    ctx.set_precision(E.Precision.fp64)
    h64, s64 = ctx.hals_solve(g, c, h0, sweeps, 1e-300)
    ctx.set_precision(E.Precision.tf32)
    h32, s32 = ctx.hals_solve(g, c, h0, sweeps, 1e-300)
    ctx.close()
    assert s64 == sweeps and s32 == sweeps
    assert np.all(np.isfinite(h32)) and h32.min() >= 0.0
    f64, f32 = _objective(g, c, h64), _objective(g, c, h32)
    # the decrease of the objective from the start agrees within 2e-4 of itself
    assert abs(f32 - f64) <= 2e-4 * abs(f64 - f0), (f0, f64, f32)
    # one more FP64 sweep from the TF32 result does not move it (it is a near-stationary point of
    # the same problem, not of a perturbed one)
    ctx = E.Context(0)
    h_ref, _ = ctx.hals_solve(g, c, h64, 1, 1e-300)
    h_pol, _ = ctx.hals_solve(g, c, h32, 1, 1e-300)
    ctx.close()
    step64 = np.max(np.abs(h_ref - h64))
    step32 = np.max(np.abs(h_pol - h32))
    assert step32 <= max(20.0 * step64, 2e-2 * np.max(h64)), (step32, step64)

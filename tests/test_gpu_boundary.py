"""GPU tier: the drop-in boundary and the reference's failure contract.

* The C++ namespace swap (include/enmf_gpu.hpp): examples/dropin_run.cpp, compiled against the
  UNMODIFIED reference headers (engine.hpp:447-449's enmf::run vs enmf::gpu::run on config 1),
  run as a separate process.  The binary is built by __graft_entry__.build() where
  /root/reference exists and travels with the repository (like libenmf_gpu.so).
* NonFiniteIterate (engine.hpp:334-337): X near the top of the FP64 range makes W_yᵀX overflow,
  the H update produces +inf, and the reference throws at iteration 1; the device flags it in
  the same iteration and the step API (begin/step/sync) reports ENMF_NON_FINITE — for the
  bitwise-order path and the product path alike — and the context stays usable.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_1805_06604_b200 as E

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "examples", "dropin_run")


def test_cpp_namespace_swap_dropin():
    if not os.path.exists(DROPIN):
        if os.path.isdir("/root/reference/proj/include"):
            subprocess.run(["make", "-C", os.path.join(ROOT, "examples")], check=True)
        else:
            pytest.skip("examples/dropin_run not built (needs the reference headers at build time)")
    res = subprocess.run([DROPIN], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "restart mismatches 0" in res.stdout, res.stdout


def _overflow_case():
    rng = np.random.default_rng(1)
    return rng.random((40, 30)) * 1.5e308, rng.random((40, 4)), rng.random((4, 30))


@pytest.mark.parametrize("prec", [E.Precision.fp64, E.Precision.fp64_exact])
def test_non_finite_iterate_through_step_api(ctx, prec):
    x, w0, h0 = _overflow_case()
    c = E.algorithm_config("e-ahals-hp3")
    c.max_outer_iterations = 5
    c.precision = prec
    ctx.load(x)
    ctx.begin(w0, h0, c)
    ctx.step(5)
    with pytest.raises(E.NonFiniteIterate):
        ctx.sync()
    try:
        ctx.end()
    except E.NonFiniteIterate:
        pass
    # the one-call entry raises the same, and the context keeps working afterwards
    with pytest.raises(E.NonFiniteIterate):
        ctx.run(x, w0, h0, c, E.TimingMode.none)
    rec = ctx.run(x * 1e-300, w0, h0, c, E.TimingMode.none)
    assert len(rec.iterations) == 6 and np.all(np.isfinite(rec.factors.w))


def test_non_finite_data_matrix_rejected(ctx):
    """DenseMatrix rejects NaN/Inf (matrix.hpp:43-51): enmf_gpu_load_dense fails at once;
    enmf_gpu_run_dense — whose upload of X overlaps begin() — fails the call with the same error
    at its first synchronization, and the context keeps working."""
    rng = np.random.default_rng(3)
    x, w0, h0 = rng.random((70, 50)), rng.random((70, 5)), rng.random((5, 50))
    c = E.algorithm_config("e-ahals-hp3")
    c.max_outer_iterations = 4
    good = ctx.run(x, w0, h0, c, E.TimingMode.none)
    for bad_value in (np.nan, np.inf):
        xb = x.copy()
        xb[13, 7] = bad_value
        with pytest.raises(E.InvalidArgument, match="DenseMatrix: values must be finite"):
            ctx.load(xb)
        with pytest.raises(E.InvalidArgument, match="DenseMatrix: values must be finite"):
            ctx.run(xb, w0, h0, c, E.TimingMode.none)
    again = ctx.run(x, w0, h0, c, E.TimingMode.none)
    assert np.array_equal(again.column("error"), good.column("error"))
    assert np.array_equal(again.factors.w, good.factors.w)

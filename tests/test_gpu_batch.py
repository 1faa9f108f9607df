"""GPU tier: the packed many-small-runs backend (csrc/batch.cuh — one CTA per run, one launch
per batch; the paper protocol's run grid, bench.hpp:233-294) against the oracle, through the
C-ABI (enmf_gpu_run_batch_dense).  Bars as for every FP64 product path (BASELINE.json
north_star): identical restart sequence, per-iteration errors within 1e-9 relative, final
factors within 1e-6, and identical inner sweep counts."""
import numpy as np
import pytest

import paper_1805_06604_b200 as E
from oracle.oracle import preset
from test_gpu_parity import _cfg, _cfg_from_meta, assert_parity

pytestmark = pytest.mark.gpu


def _check_run(rec, ref, kappa=False):
    assert_parity(rec, ref[0]["error"], ref[0]["restarted"], ref[1], ref[2], ref[3], kappa=kappa)
    if not kappa:   # below the noise floor (noise-free E-ANLS) BPP's rounds follow rounding noise
        assert np.array_equal(rec.column("inner_h_count"), ref[0]["inner_h"])
        assert np.array_equal(rec.column("inner_w_count"), ref[0]["inner_w"])


@pytest.mark.parametrize("alg", ["e-ahals-hp3", "e-ahals-hp1", "ahals", "e-anls-hp1", "e-anls-hp3", "anls"])
def test_c1_batch_vs_oracle(port, golden, alg):
    """Config 1 (200 × 200, r = 20, 200 outer iterations) for 24 initialisations in one launch,
    every preset of the protocol (E-ANLS: BPP inner solves; on this noise-free data its error
    reaches ~5e-7·||X||, so the per-iteration bar includes the trace identity's own
    cancellation bound, as in test_gpu_parity.test_c1_fp64_parity_vs_reference)."""
    x = golden.load("c1_inputs")["x"]
    probs = []
    for s in range(24):
        w0, h0 = port.random_init(200, 200, 20, 100 + s)
        probs.append((x, w0, h0))
    cfg = _cfg(alg, 200)
    out = E.run_batch(probs, cfg, backend="packed")
    for (xx, w0, h0), rec in zip(probs[::5], out[::5]):          # every 5th run vs the oracle
        ref = port.run_dense(xx, w0, h0, preset(alg, max_outer_iterations=200))
        _check_run(rec, ref, kappa="anls" in alg)


@pytest.mark.parametrize("variant", [dict(hp=2), dict(hp=1, literal_hp1_order=True),
                                     dict(extrapolation_enabled=False), dict(beta0=0.0),
                                     dict(inner_max_sweeps=3)])
def test_config_variants_vs_oracle(port, golden, variant):
    """hp 2, literal hp1, extrapolation off, β0 = 0, forced sweep counts (engine.hpp:309-440)."""
    x = golden.load("c1_inputs")["x"]
    w0, h0 = port.random_init(200, 200, 20, 7)
    cfg = _cfg("e-ahals-hp3", 60, **variant)
    rec = E.run_batch_packed([(x, w0, h0)], cfg)[0]
    kw = dict(variant)
    if "inner_max_sweeps" in kw:
        kw["inner_max_sweeps"] = kw["inner_max_sweeps"]
    ref = port.run_dense(x, w0, h0, preset("e-ahals-hp3", max_outer_iterations=60, **kw))
    _check_run(rec, ref)


@pytest.mark.parametrize("alg", ["e-ahals-hp3", "e-anls-hp1"])
@pytest.mark.parametrize("shape", [(150, 260, 13), (280, 40, 32), (37, 301, 1), (64, 280, 32), (90, 113, 7)])
def test_shapes_vs_oracle(port, shape, alg):
    """Ragged shapes: n > 256 columns per CTA (thread loops), r = 1 and the r = 32 maximum."""
    m, n, r = shape
    rng = np.random.default_rng(m + n + r)
    x = rng.random((m, r)) @ rng.random((r, n)) + np.abs(0.01 * rng.standard_normal((m, n)))
    probs = [(x, *port.random_init(m, n, r, s)) for s in (3, 4, 5)]
    # r = 1 converges within ~5 iterations; past that the errors tie to the last bit and the
    # restart decisions are rounding noise in any summation order
    it = 4 if r == 1 else 40
    out = E.run_batch_packed(probs, _cfg(alg, it))
    for (xx, w0, h0), rec in zip(probs, out):
        _check_run(rec, port.run_dense(xx, w0, h0, preset(alg, max_outer_iterations=it)))


def test_dead_column_reinit(golden):
    """gram_with_reinit (engine.hpp:268-296) inside the packed kernel: the reference's redraw."""
    inp = golden.load("reinit_inputs")
    g = golden.load("reinit_hals")
    cfg = _cfg_from_meta(golden.meta["reinit_hals"], E.Precision.fp64)
    rec = E.run_batch_packed([(inp["x"], inp["w0"], inp["h0"])] * 3, cfg)
    for r in rec:
        assert r.iterations[1].reinit_events & 1
        assert_parity(r, g["error"], g["restarted"], g["w"], g["h"], float(g["norm_x"]))


def test_batch_matches_itself_across_grid_sizes(port, golden):
    """A run's result does not depend on the batch it is in (1 run vs 400 runs: several runs per
    CTA, every SM busy): bitwise."""
    x = golden.load("c1_inputs")["x"]
    probs = [(x, *port.random_init(200, 200, 20, 500 + s)) for s in range(400)]
    cfg = _cfg("e-ahals-hp3", 50)
    big = E.run_batch_packed(probs, cfg)
    for i in (0, 137, 399):
        one = E.run_batch_packed([probs[i]], cfg)[0]
        assert np.array_equal(one.column("error"), big[i].column("error"))
        assert np.array_equal(one.factors.w, big[i].factors.w) and np.array_equal(one.factors.h, big[i].factors.h)


def test_eligibility_and_errors(golden):
    x = golden.load("c1_inputs")["x"]
    rng = np.random.default_rng(1)
    assert E.batch_eligible(200, 200, 20, _cfg("e-ahals-hp3", 10))
    assert not E.batch_eligible(200, 200, 33, _cfg("e-ahals-hp3", 10))                 # r > 32
    assert E.batch_eligible(200, 200, 20, _cfg("e-anls-hp1", 10))                      # BPP, r <= 32
    assert not E.batch_eligible(200, 200, 20, _cfg("e-ahals-hp3", 10, E.Precision.fp64_exact))
    with pytest.raises(E.InvalidArgument):
        E.run_batch([(x, rng.random((200, 33)), rng.random((33, 200)))], _cfg("e-ahals-hp3", 5), backend="packed")
    with pytest.raises(E.InvalidArgument):                                               # negative init
        E.run_batch_packed([(x, -rng.random((200, 20)), rng.random((20, 200)))], _cfg("e-ahals-hp3", 5))
    # auto picks the streams backend for fp64_exact and stays bitwise there
    p = (x, rng.random((200, 20)), rng.random((20, 200)))
    cfg = _cfg("e-anls-hp1", 3, E.Precision.fp64_exact)
    out = E.run_batch([p], cfg)
    one = E.Context().run(*p, cfg, E.TimingMode.none)
    assert np.array_equal(out[0].column("error"), one.column("error"))


def test_failing_run_is_reported_per_run(golden, port):
    """A run whose H update overflows (a column of X at 1e307: W_yᵀX is +inf) fails with
    NonFiniteIterate (engine.hpp:334-337, "H update produced a non-finite value", as the reference
    does for this input) in its own slot; the other runs of the launch finish."""
    x = golden.load("c1_inputs")["x"]
    bad = x.copy()
    bad[:, 0] = 1e307
    w0, h0 = port.random_init(200, 200, 20, 3)
    cfg = _cfg("e-ahals-hp3", 10)
    out = E.run_batch_packed([(x, w0, h0), (bad, w0, h0), (x, w0, h0)], cfg, raise_errors=False)
    assert isinstance(out[1], E.NonFiniteIterate)
    assert not isinstance(out[0], Exception) and not isinstance(out[2], Exception)
    assert np.array_equal(out[0].column("error"), out[2].column("error"))
    with pytest.raises(E.NonFiniteIterate):
        E.run_batch_packed([(bad, w0, h0)], cfg)
    with pytest.raises(E.NonFiniteIterate):                       # the single-run engine agrees
        E.Context().run(bad, w0, h0, cfg, E.TimingMode.none)

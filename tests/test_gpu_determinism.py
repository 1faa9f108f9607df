"""Race detection without compute-sanitizer (closed on this GPU pool): the hand-rolled
synchronisation — the persistent sweep kernels' grid-wide arrive/epoch protocol, speculative
stall decision and named-barrier / TMEM hand-offs (hals.cuh, hals_tm.cuh), BPP's warp-level
exchanges, the tcgen05 digit GEMM's mbarrier pipeline (ozk.cuh), the sharded engine's
peer-memory mailboxes (dist.cuh) — is deterministic by construction (fixed-order sums, no
atomics on data).  A race shows up as run-to-run differences, so every family is run
repeatedly, also with other work in flight on concurrent streams (run_batch) to shift the
CTAs' relative timing, and must reproduce its records and factors bit for bit."""
import numpy as np
import pytest

import paper_1805_06604_b200 as E

pytestmark = pytest.mark.gpu


def _problem(m, n, r, seed):
    rng = np.random.default_rng(seed)
    x = rng.random((m, r)) @ rng.random((r, n)) + np.abs(0.01 * rng.standard_normal((m, n)))
    return x, rng.random((m, r)), rng.random((r, n))


def _cfg(alg, it):
    c = E.algorithm_config(alg)
    c.max_outer_iterations = it
    return c


def _same(a, b):
    assert np.array_equal(a.column("error"), b.column("error"))
    assert np.array_equal(a.column("inner_h_count"), b.column("inner_h_count"))
    assert np.array_equal(a.column("inner_w_count"), b.column("inner_w_count"))
    assert np.array_equal(a.factors.w, b.factors.w) and np.array_equal(a.factors.h, b.factors.h)


@pytest.mark.parametrize("shape,alg,reps", [((300, 260, 20), "e-ahals-hp3", 12),     # sweep_ws
                                            ((700, 3000, 100), "e-ahals-hp3", 8),    # sweep_tm
                                            ((256, 40000, 128), "e-ahals-hp3", 3),   # sweep_tm, two rounds
                                            ((400, 380, 20), "e-anls-hp1", 8),       # BPP
                                            ((4096, 4096, 16), "e-ahals-hp3", 3)])   # INT8-digit products
def test_repeated_runs_bitwise(ctx, shape, alg, reps):
    x, w0, h0 = _problem(*shape, seed=sum(shape))
    cfg = _cfg(alg, 8)
    first = ctx.run(x, w0, h0, cfg, E.TimingMode.none)
    for _ in range(reps - 1):
        _same(first, ctx.run(x, w0, h0, cfg, E.TimingMode.none))


@pytest.mark.parametrize("shape", [(700, 3000, 100), (4096, 4096, 128)])
def test_tf32_variant_repeated_runs_bitwise(ctx, shape):
    """The TF32 variant's tcgen05 kernels — the right-looking sweeps with the residual in tensor
    memory (hals_rl.cuh: TMEM stores → TS-form MMA → mbarrier → TMEM loads, two column groups per
    CTA on their own barriers) and, at 4096², the kind::tf32 cross-product GEMM — reproduce their
    records and factors bit for bit."""
    x, w0, h0 = _problem(*shape, seed=sum(shape) + 1)
    cfg = _cfg("e-ahals-hp3", 8)
    cfg.precision = E.Precision.tf32
    first = ctx.run(x, w0, h0, cfg, E.TimingMode.none)
    assert first.column("inner_h_count")[1:].min() >= 1
    for _ in range(5):
        _same(first, ctx.run(x, w0, h0, cfg, E.TimingMode.none))


def test_concurrent_streams_bitwise(ctx):
    """The same problems run alone and as a batch on 4 concurrent streams (persistent sweep
    kernels sharing the SMs with other graphs' kernels): identical results."""
    probs = [_problem(500, 2100, 100, 11 + i) for i in range(3)] + [_problem(300, 260, 20, 20 + i) for i in range(3)]
    cfg = _cfg("e-ahals-hp3", 6)
    alone = [ctx.run(x, w, h, cfg, E.TimingMode.none) for x, w, h in probs]
    for rep in range(2):
        batch = E.run_batch(probs, cfg, streams=4, backend="streams")
        for a, b in zip(alone, batch):
            _same(a, b)


def test_sharded_world1_repeated_bitwise():
    """The sharded engine at world 1 (every exchange kernel: all-gathers, mailbox all-reduces,
    per-sweep gain exchange) reproduces itself bit for bit."""
    from paper_1805_06604_b200.dist import ShardedContext
    m, n, r = 260, 300, 20
    x, w0, h0 = _problem(m, n, r, 3)
    outs = []
    for _ in range(4):
        sc = ShardedContext(0, 0, 1, m, n, r, lambda b: [b])
        try:
            cfg = _cfg("e-ahals-hp3", 6)
            sc.load_sharded(*sc.shard_x(x))
            sc.begin(w0, h0, cfg)
            sc.step(6)
            recs = sc.sync()
            w = np.empty((m, r))
            h = np.empty((r, n))
            sc.end(w.ctypes.data, h.ctypes.data)
        finally:
            sc.finalize()
        outs.append((np.array([it.error for it in recs]), w, h))
    for e, w, h in outs[1:]:
        assert np.array_equal(e, outs[0][0]) and np.array_equal(w, outs[0][1]) and np.array_equal(h, outs[0][2])

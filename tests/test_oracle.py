"""CPU tier: the oracle restatement pinned against the reference.

(1) against the committed golden fixtures produced by the reference itself
    (tests/golden/make_golden.py, via oracle/_ref), and the SURVEY/BASELINE
    known answers;  (2) against oracle/_ref directly (bitwise) where it exists.
"""
import numpy as np
import pytest

from oracle.oracle import OracleError, default_config, preset

PRESETS = ["e-ahals-hp3", "e-ahals-hp1", "e-anls-hp1", "anls", "ahals", "e-anls-hp3"]


def _cfg_from_meta(meta):
    c = default_config()
    for k, v in meta.items():
        if hasattr(c, k) and k not in ("final_relative_error", "restarts"):
            setattr(c, k, v)
    return c


@pytest.mark.parametrize("name", PRESETS)
def test_port_matches_reference_golden_c1(port, golden, name):
    inp = golden.load("c1_inputs")
    g = golden.load(f"c1_{name}")
    rec, w, h, nx = port.run_dense(inp["x"], inp["w0"], inp["h0"], preset(name, max_outer_iterations=200))
    assert np.array_equal(rec["error"], g["error"])
    assert np.array_equal(rec["restarted"], g["restarted"])
    assert np.array_equal(rec["beta"], g["beta"])
    assert np.array_equal(w, g["w"]) and np.array_equal(h, g["h"])
    assert nx == float(g["norm_x"])


def test_known_answers(port, golden):
    """SURVEY.md §6.2 / BASELINE.md §2: config-1 final relative errors, 5 restarts each."""
    ka = golden.meta["known_answers"]
    inp = golden.load("c1_inputs")
    for name, key in (("e-ahals-hp3", "c1_e-ahals-hp3_final_relative_error"),
                      ("e-ahals-hp1", "c1_e-ahals-hp1_final_relative_error")):
        rec, *_ = port.run_dense(inp["x"], inp["w0"], inp["h0"], preset(name, max_outer_iterations=200))
        assert rec["relative_error"][-1] == ka[key]
        assert rec["restarted"].sum() == ka["c1_restarts"]


def test_generators_match_reference_streams(port, golden):
    inp = golden.load("c1_inputs")
    assert np.array_equal(port.gen_lowrank(200, 200, 20, 1), inp["x"])
    w, h = port.random_init(200, 200, 20, 2)
    assert np.array_equal(w, inp["w0"]) and np.array_equal(h, inp["h0"])


@pytest.mark.parametrize("tag", ["small_hals_hp2", "small_hals_hp1_literal", "small_exact_hp2",
                                 "small_exact_hp1_literal", "small_hals_noextrap", "small_hals_beta0",
                                 "small_mixed_hals_exact", "small_hals_sweeps3"])
def test_port_variants_golden(port, golden, tag):
    inp = golden.load("small_inputs")
    g = golden.load(tag)
    cfg = _cfg_from_meta(golden.meta[tag])
    rec, w, h, _ = port.run_dense(inp["x"], inp["w0"], inp["h0"], cfg)
    assert np.array_equal(rec["error"], g["error"])
    assert np.array_equal(rec["restarted"], g["restarted"])
    assert np.array_equal(w, g["w"]) and np.array_equal(h, g["h"])


@pytest.mark.parametrize("tag", ["reinit_hals", "reinit_exact"])
def test_port_reinit_golden(port, golden, tag):
    """Dead starting column -> deterministic redraw (engine.hpp:268-296)."""
    inp = golden.load("reinit_inputs")
    g = golden.load(tag)
    rec, w, h, _ = port.run_dense(inp["x"], inp["w0"], inp["h0"], _cfg_from_meta(golden.meta[tag]))
    assert rec["reinit"][1] & 1, "the W_y reinit must fire at iteration 1"
    assert np.array_equal(rec["error"], g["error"])
    assert np.array_equal(w, g["w"]) and np.array_equal(h, g["h"])


def test_kernels_golden(port, golden):
    k = golden.load("kernels")
    assert np.array_equal(port.gram(k["w"]), k["gram"])
    assert np.array_equal(port.cross_wx(k["w"], k["x"]), k["cross"])
    hh, _ = port.hals_solve(k["gram"], k["cross"], k["h0"], 25, 0.01)
    assert np.array_equal(hh, k["hals"])
    ha, _ = port.active_set_solve(k["gram"], k["cross"], np.abs(k["h0"]))
    assert np.array_equal(ha, k["bpp"])


def test_gram_bitwise_symmetric(port):
    a = np.random.default_rng(3).random((57, 9))
    g = port.gram(a)
    assert np.array_equal(g, g.T)


def test_update_beta_worked_transitions(port):
    """acceptance.cpp:340-372 / test_engine.cpp:154-195: exact equality."""
    t1 = port.update_beta(dict(beta=0.5, beta_bar=1.0, beta_prev=0.5, gamma=1.1, gamma_bar=1.05, eta=1.5), True)
    assert t1["beta"] == min(1.0, 1.1 * 0.5) and t1["beta_bar"] == 1.0
    t2 = port.update_beta(dict(beta=0.6, beta_bar=0.6, beta_prev=0.5, gamma=1.1, gamma_bar=1.05, eta=1.5), True)
    assert t2["beta"] == 0.6 and t2["beta_bar"] == min(1.0, 1.05 * 0.6)
    t3 = port.update_beta(dict(beta=0.6, beta_bar=1.0, beta_prev=0.5, gamma=1.1, gamma_bar=1.05, eta=1.5), False)
    assert t3["beta"] == 0.6 / 1.5 and t3["beta_bar"] == 0.5
    s4 = dict(beta=0.0, beta_bar=1.0, beta_prev=0.0, gamma=1.1, gamma_bar=1.05, eta=1.5)
    assert port.update_beta(s4, True)["beta"] == 0.0 and port.update_beta(s4, False)["beta"] == 0.0


def test_bpp_matches_enumeration(port):
    """nnls.hpp active_set_solve == exhaustive 2^r passive-set search (oracles.hpp:141-188)."""
    rng = np.random.default_rng(31)
    for inst in range(40):
        r = int(rng.integers(1, 6))
        m = r + int(rng.integers(0, 8))
        w = rng.random((m, r))
        x = rng.random((m, 4)) * (1 if inst % 2 else 2) - (0 if inst % 2 else 1)
        G, Cm = w.T @ w, w.T @ x
        h, _ = port.active_set_solve(G, Cm, np.zeros((r, 4)))
        for col in range(4):
            best, bestv = None, np.inf
            for mask in range(1 << r):
                idx = [i for i in range(r) if mask >> i & 1]
                v = np.zeros(r)
                if idx:
                    try:
                        sol = np.linalg.solve(G[np.ix_(idx, idx)], Cm[idx, col])
                    except np.linalg.LinAlgError:
                        continue
                    if np.any(sol < -1e-12):
                        continue
                    v[idx] = np.maximum(sol, 0)
                obj = 0.5 * v @ G @ v - Cm[:, col] @ v
                if obj < bestv:
                    bestv, best = obj, v
            got = 0.5 * h[:, col] @ G @ h[:, col] - Cm[:, col] @ h[:, col]
            assert abs(got - bestv) <= 1e-9 * (1 + abs(bestv))


def test_config_validation(port):
    bad = [dict(hp=4), dict(beta0=1.0), dict(beta0=-0.1), dict(gamma=1.01, gamma_bar=1.05),
           dict(max_seconds=0.0), dict(inner_sweep_ratio=0.0), dict(inner_stall_fraction=1.0)]
    x = np.random.default_rng(0).random((6, 5))
    w, h = port.random_init(6, 5, 2, 1)
    for kw in bad:
        with pytest.raises(OracleError) as e:
            port.run_dense(x, w, h, default_config(max_outer_iterations=1, **kw))
        assert e.value.code == 1


def test_rejects_negative_init(port):
    x = np.random.default_rng(0).random((6, 5))
    w, h = port.random_init(6, 5, 2, 1)
    w[0, 0] = -1e-3
    with pytest.raises(OracleError):
        port.run_dense(x, w, h, default_config(max_outer_iterations=1))


def test_empty_budget(port):
    x = np.random.default_rng(0).random((6, 5))
    w, h = port.random_init(6, 5, 2, 1)
    rec, w1, h1, _ = port.run_dense(x, w, h, default_config(max_outer_iterations=0))
    assert len(rec["error"]) == 1 and np.array_equal(w1, w) and np.array_equal(h1, h)


# ---- against the compiled reference directly (only where oracle/_ref exists)
@pytest.mark.parametrize("seed", range(6))
def test_port_bitwise_vs_reference_random(port, ref, seed):
    rng = np.random.default_rng(seed)
    m, n, r = (int(v) for v in rng.integers(4, 40, 3))
    r = max(1, min(r % 9 + 1, m, n))
    x = rng.random((m, n))
    w0, h0 = port.random_init(m, n, r, seed + 10)
    for name in PRESETS:
        cfg = preset(name, max_outer_iterations=25, reinit_seed=seed)
        a, b = port.run_dense(x, w0, h0, cfg), ref.run_dense(x, w0, h0, cfg)
        assert np.array_equal(a[0]["error"], b[0]["error"]), name
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]), name


def test_port_csr_vs_reference(port, ref):
    off, cidx, vals = port.gen_docs(300, 120, 4)
    m, n, r = 300, 120, 6
    w0, h0 = port.random_init(m, n, r, 9)
    cfg = preset("e-ahals-hp3", max_outer_iterations=15)
    a = port.run_csr(off, cidx, vals, m, n, w0, h0, cfg)
    b = ref.run_csr(off, cidx, vals, m, n, w0, h0, cfg)
    assert np.array_equal(a[0]["error"], b[0]["error"])
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("name", ["e-ahals-hp3", "e-anls-hp1"])
def test_port_csr_vs_golden(port, golden, name):
    """The C restatement's CSR path is bitwise the reference's (fixtures from the reference)."""
    inp = golden.load("csr_inputs")
    g = golden.load(f"csr_{name}")
    rec, w, h, nx = port.run_csr(inp["off"], inp["cidx"], inp["vals"], int(inp["m"]), int(inp["n"]),
                                 inp["w0"], inp["h0"], preset(name, max_outer_iterations=40))
    assert np.array_equal(rec["error"], g["error"])
    assert np.array_equal(rec["restarted"].astype(np.int32), g["restarted"].astype(np.int32))
    assert np.array_equal(w, g["w"]) and np.array_equal(h, g["h"]) and nx == float(g["norm_x"])


# ------------------------------------------------ the multi-threaded replica (replica.c)
def _replica(port, threads, fn):
    old = port.threads
    port.threads = threads
    try:
        return fn()
    finally:
        port.threads = old


def _same(a, b, counts=False):
    """Bitwise-equal runs; counts: also the sweep / BPP counts (the reference's IterationRecord has
    none, engine.hpp:216-223 — oracle/_ref reports zeros)."""
    keys = ("error", "beta", "restarted") + (("inner_h", "inner_w") if counts else ())
    return (all(np.array_equal(a[0][k], b[0][k]) for k in keys)
            and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and a[3] == b[3])


@pytest.mark.parametrize("name", ["e-ahals-hp3", "e-ahals-hp1", "e-anls-hp1", "ahals"])
def test_replica_bitwise_vs_reference_golden_c1(port, golden, name):
    """The replica (oracle/replica.c, 4 threads) reproduces the reference's own C1 fixtures bit for bit."""
    inp = golden.load("c1_inputs")
    g = golden.load(f"c1_{name}")
    rec, w, h, nx = _replica(port, 4, lambda: port.run_dense(inp["x"], inp["w0"], inp["h0"],
                                                             preset(name, max_outer_iterations=200)))
    assert np.array_equal(rec["error"], g["error"]) and np.array_equal(rec["beta"], g["beta"])
    assert np.array_equal(w, g["w"]) and np.array_equal(h, g["h"]) and nx == float(g["norm_x"])


@pytest.mark.parametrize("shape", [(301, 257, 17), (517, 1303, 72), (1000, 777, 33), (64, 1000, 5), (130, 70, 128)])
def test_replica_bitwise_vs_reference(port, ref, shape):
    """Ragged shapes (tails of every vector block, r > the column block) vs oracle/_ref, bitwise."""
    m, n, r = shape
    rng = np.random.default_rng(m)
    x = rng.random((m, r)) @ rng.random((r, n)) + np.abs(0.01 * rng.standard_normal((m, n)))
    w0, h0 = port.random_init(m, n, r, 3)
    cfg = preset("e-ahals-hp3", max_outer_iterations=12)
    assert _same(_replica(port, 8, lambda: port.run_dense(x, w0, h0, cfg)), ref.run_dense(x, w0, h0, cfg))


def test_replica_bitwise_vs_port_thread_counts(port):
    """Any thread count gives the single-threaded port's bits (C2-shaped case, 15 iterations)."""
    x = port.gen_config(2, 2000, 300, 24, 1)
    w0, h0 = port.random_init(2000, 300, 24, 2)
    cfg = preset("e-ahals-hp3", max_outer_iterations=15)
    base = port.run_dense(x, w0, h0, cfg)
    for t in (2, 3, 8):
        assert _same(_replica(port, t, lambda: port.run_dense(x, w0, h0, cfg)), base, counts=True), t


def test_tiled_generator_thread_independent(port):
    """orc_gen_tiled: per-tile streams, identical bits for any thread count and tile-aligned blocks."""
    a = port.gen_tiled(700, 900, 8, 5, tile=256, threads=1)
    b = port.gen_tiled(700, 900, 8, 5, tile=256, threads=7)
    assert np.array_equal(a, b)
    assert np.all(a > 0) and a.shape == (700, 900)


def test_product_tiled_generator_matches_oracle(port):
    """The product's C5 data generator (csrc/io.cpp enmf_gen_tiled, used by bench.py's GPU arm)
    draws the oracle's streams bit for bit, whole matrix and rank blocks alike."""
    from paper_1805_06604_b200 import data
    m, n, r, T = 700, 900, 8, 256
    full = port.gen_tiled(m, n, r, 5, tile=T, threads=3)
    assert np.array_equal(data.gen_tiled(m, n, r, 5, tile=T), full)
    assert np.array_equal(data.gen_tiled(m, n, r, 5, rows=slice(256, 700), tile=T), full[256:])
    assert np.array_equal(data.gen_tiled(m, n, r, 5, cols=slice(100, 613), tile=T), full[:, 100:613])


def test_reference_raises_non_finite_on_overflow(port, ref):
    """The NonFiniteIterate case of tests/test_gpu_boundary.py: X near the top of the FP64 range,
    W_yᵀX overflows, the reference throws in iteration 1 (engine.hpp:334-337) — port and reference."""
    rng = np.random.default_rng(1)
    x, w0, h0 = rng.random((40, 30)) * 1.5e308, rng.random((40, 4)), rng.random((4, 30))
    for o in (port, ref):
        with pytest.raises(OracleError, match="non-finite"):
            o.run_dense(x, w0, h0, preset("e-ahals-hp3", max_outer_iterations=5))

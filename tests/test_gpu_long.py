"""GPU tier: full-length BASELINE configs against the reference's own trajectories.

Fixtures (tests/golden/long_*.npz, made by tests/golden/make_golden_long.py):
  * C2 10304×400 r=40 E-A-HALS hp3, 500 iterations;  C3 2000² r=30 E-ANLS hp1, 100;
    C4 30000×10000 CSR r=20 E-A-HALS hp3, 300 — the unmodified reference (`enmf::run`,
    engine.hpp:447-521, compiled in place);
  * C5 32768² r=128 E-A-HALS hp3, 25 iterations — the bit-exact multi-threaded replica
    (oracle/replica.c), itself pinned bitwise to the reference (tests/test_oracle.py and
    golden_long.json "c5check": C5 iteration 1).
The inputs are regenerated here from their seeds with the C generators (oracle/liboracle.so);
‖X‖ doubles as the checksum that the regenerated X is the one the fixture was made from.

Bars (north_star, FP64 product mode — at C5 the INT8-digit cross products on the tensor cores):
identical restart sequence and inner sweep counts, per-iteration e/‖X‖ within 1e-9 relative,
final W, H within 1e-6 (whole factors for C2/C3; seeded 4096-entry samples and per-component
norms for C4/C5).
"""
import json
import os
import sys

import numpy as np
import pytest

import paper_1805_06604_b200 as E

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, GOLDEN)
from make_golden_long import CONFIGS, factor_summary, inputs  # noqa: E402

pytestmark = pytest.mark.gpu

REL_ERR_TOL = 1e-9
FACTOR_TOL = 1e-6


def _load(tag):
    path = os.path.join(GOLDEN, f"long_{tag}.npz")
    if not os.path.exists(path):
        pytest.fail(f"fixture {path} missing (tests/golden/make_golden_long.py {tag})")
    return dict(np.load(path))


def _cfg(name, iters):
    c = E.algorithm_config(name)
    c.max_outer_iterations = iters
    return c


def check(rec, g, w, h, whole):
    """north_star bars against a long fixture; returns the max relative error deviation."""
    err = rec.column("error")
    assert len(err) == len(g["error"])
    assert np.array_equal(rec.column("restarted").astype(np.int32), g["restarted"].astype(np.int32)), \
        "restart sequence differs"
    assert np.array_equal(rec.column("inner_h_count"), g["inner_h"]), "H-side sweep / BPP counts differ"
    assert np.array_equal(rec.column("inner_w_count"), g["inner_w"]), "W-side sweep / BPP counts differ"
    assert np.array_equal(rec.column("beta"), g["beta"]), "β sequence differs"
    dev = np.abs(err - g["error"]) / g["error"]
    assert np.all(dev <= REL_ERR_TOL), f"max relative error deviation {dev.max():.3e} at k={int(dev.argmax())}"
    if whole:
        assert np.max(np.abs(w - g["w"])) <= FACTOR_TOL * np.max(np.abs(g["w"]))
        assert np.max(np.abs(h - g["h"])) <= FACTOR_TOL * np.max(np.abs(g["h"]))
    s = factor_summary(w, h)
    for k in ("w_sample", "h_sample"):
        assert np.max(np.abs(s[k] - g[k])) <= FACTOR_TOL * np.max(np.abs(g[k])), k
    for k in ("w_colnorm", "h_rownorm"):
        assert np.max(np.abs(s[k] - g[k]) / g[k]) <= FACTOR_TOL, k
    return float(dev.max())


@pytest.mark.parametrize("tag", ["c2", "c3"])
def test_dense_configs_full_length(ctx, port, tag):
    """C2 (500 iterations) and C3 (100, E-ANLS: block principal pivoting both sides)."""
    c = CONFIGS[tag]
    g = _load(tag)
    x, w0, h0 = inputs(port, c)
    rec = ctx.run(x, w0, h0, _cfg(c["alg"], c["iters"]), E.TimingMode.none)
    assert abs(rec.norm_x - float(g["norm_x"])) <= 1e-14 * float(g["norm_x"]), "regenerated X differs"
    check(rec, g, rec.factors.w, rec.factors.h, whole=True)


def test_c4_csr_full_length(ctx, port):
    """C4: 30000×10000 document-shaped CSR (≈1.3 M nnz), r=20, 300 iterations."""
    c = CONFIGS["c4"]
    g = _load("c4")
    (off, cidx, vals), w0, h0 = inputs(port, c)
    rec = ctx.run_csr(off, cidx, vals, c["m"], c["n"], w0, h0, _cfg(c["alg"], c["iters"]), E.TimingMode.none)
    assert abs(rec.norm_x - float(g["norm_x"])) <= 1e-14 * float(g["norm_x"])
    check(rec, g, rec.factors.w, rec.factors.h, whole=False)


def test_c5_headline_config_vs_replica(ctx, port):
    """C5 itself (m = n = 32768, r = 128, E-A-HALS hp3 — the benchmarked configuration) for 25
    outer iterations through the product path (INT8-digit cross products, persistent DMMA
    sweeps with up to 129 sweeps per update) against the replica's trajectory."""
    c = CONFIGS["c5"]
    g = _load("c5")
    x, w0, h0 = inputs(port, c)
    rec = ctx.run(x, w0, h0, _cfg(c["alg"], c["iters"]), E.TimingMode.none)
    del x
    assert abs(rec.norm_x - float(g["norm_x"])) <= 1e-14 * float(g["norm_x"]), "regenerated X differs"
    assert ctx.digit_levels[0] in (6, 7), ctx.digit_levels
    dev = check(rec, g, rec.factors.w, rec.factors.h, whole=False)
    meta = json.load(open(os.path.join(GOLDEN, "golden_long.json")))
    print(f"C5 vs replica: max rel error deviation {dev:.3e}; sweeps {meta['c5']['sweeps_h'][-3:]}")

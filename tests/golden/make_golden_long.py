"""Full-length golden trajectories for BASELINE configs 2-5 (VERDICT r01 "next round" #1).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden_long.py c2 c3 c4     # the reference itself (oracle/_ref)
    python tests/golden/make_golden_long.py c5           # the bit-exact multi-threaded replica
    python tests/golden/make_golden_long.py c5check      # replica vs the reference, C5 iteration 1

* C2 (10304×400 r=40, E-A-HALS hp3, 500 iterations), C3 (2000² r=30, E-ANLS hp1, 100) and
  C4 (30000×10000 CSR r=20, E-A-HALS hp3, 300) come from the UNMODIFIED reference
  (`enmf::run`, engine.hpp:447-521, compiled in place: oracle/_ref/libenmf_ref.so).
* C5 (32768² r=128, E-A-HALS hp3) would take ≈10 h single-threaded, so it comes from the
  replica (oracle/replica.c: same per-element summation order, OpenMP over independent
  elements), which tests/test_oracle.py pins bitwise to the reference on C1-C3 shapes and
  `c5check` pins on C5's first iteration.

Inputs are regenerated on the GPU box from their seeds (the generators are plain C in
oracle/liboracle.so); the fixtures store the trajectory (error, β, restart flags, sweep
counts), ‖X‖ as a checksum of the regenerated X, and the final factors — whole for the
small ones, and for C4/C5 as a seeded sample of entries plus the per-component norms.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, preset  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (generator, shape, algorithm, iterations, seeds) — BASELINE.json configs[1..4]
CONFIGS = {
    "c2": dict(kind="config", which=2, m=10304, n=400, r=40, alg="e-ahals-hp3", iters=500, seeds=(1, 2)),
    "c3": dict(kind="config", which=3, m=2000, n=2000, r=30, alg="e-anls-hp1", iters=100, seeds=(1, 2)),
    "c4": dict(kind="docs", m=30000, n=10000, r=20, alg="e-ahals-hp3", iters=300, seeds=(1, 2)),
    "c5": dict(kind="tiled", m=32768, n=32768, r=128, alg="e-ahals-hp3", iters=25, seeds=(1, 2)),
}
SAMPLE = 4096


def inputs(port, c):
    """Regenerates a config's X (dense array, or CSR triple) and W0, H0 from its seeds."""
    sd, si = c["seeds"]
    m, n, r = c["m"], c["n"], c["r"]
    if c["kind"] == "config":
        x = port.gen_config(c["which"], m, n, r, sd)
    elif c["kind"] == "docs":
        x = port.gen_docs(m, n, sd)
    else:
        x = port.gen_tiled(m, n, r, sd)
    w0, h0 = port.random_init(m, n, r, si)
    return x, w0, h0


def sample_idx(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, shape[0], SAMPLE), rng.integers(0, shape[1], SAMPLE)


def factor_summary(w, h):
    """What the fixtures keep of the final factors: seeded samples + per-component 2-norms."""
    wi, wj = sample_idx(w.shape, 101)
    hi, hj = sample_idx(h.shape, 102)
    return dict(w_sample=w[wi, wj], h_sample=h[hi, hj], w_colnorm=np.linalg.norm(w, axis=0),
                h_rownorm=np.linalg.norm(h, axis=1))


def save(tag, rec, w, h, nx, c, seconds, source, whole):
    d = dict(error=rec["error"], relative_error=rec["relative_error"], beta=rec["beta"],
             restarted=rec["restarted"], inner_h=rec["inner_h"], inner_w=rec["inner_w"],
             reinit=rec["reinit"], norm_x=nx)
    d.update(factor_summary(w, h))
    if whole:
        d.update(w=w, h=h)
    np.savez_compressed(os.path.join(OUT, f"long_{tag}.npz"), **d)
    meta_path = os.path.join(OUT, "golden_long.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    meta[tag] = dict(c, source=source, seconds=round(seconds, 1), restarts=int(rec["restarted"].sum()),
                     final_relative_error=float(rec["relative_error"][-1]),
                     sweeps_h=rec["inner_h"].tolist(), sweeps_w=rec["inner_w"].tolist())
    json.dump(meta, open(meta_path, "w"), indent=1)
    print(f"{tag}: {source} {seconds:.1f}s final rel {rec['relative_error'][-1]:.6e} "
          f"restarts {int(rec['restarted'].sum())}", flush=True)


def main(which):
    port = Oracle("port")
    for tag in which:
        if tag == "c5check":
            c5check(port)
            continue
        c = CONFIGS[tag]
        x, w0, h0 = inputs(port, c)
        cfg = preset(c["alg"], max_outer_iterations=c["iters"])
        t = time.time()
        if tag == "c5":
            port.threads = os.cpu_count()
            rec, w, h, nx = port.run_dense(x, w0, h0, cfg)
            port.threads = 1
            source = f"replica ({os.cpu_count()} threads, oracle/replica.c)"
        else:
            R = Oracle("reference")
            if c["kind"] == "docs":
                rec, w, h, nx = R.run_csr(*x, c["m"], c["n"], w0, h0, cfg)
                port.threads = 1
                p = port.run_csr(*x, c["m"], c["n"], w0, h0, cfg)
            else:
                rec, w, h, nx = R.run_dense(x, w0, h0, cfg)
                port.threads = os.cpu_count()
                p = port.run_dense(x, w0, h0, cfg)
                port.threads = 1
            # the reference's IterationRecord carries no sweep counts (engine.hpp:216-223): they come
            # from the restatement, whose trajectory must be the reference's bit for bit
            assert all(np.array_equal(p[0][k], rec[k]) for k in ("error", "beta", "restarted"))
            assert np.array_equal(p[1], w) and np.array_equal(p[2], h) and p[3] == nx
            rec["inner_h"], rec["inner_w"] = p[0]["inner_h"], p[0]["inner_w"]
            source = "reference (oracle/_ref, enmf::run); sweep counts from the bitwise-equal port"
        save(tag, rec, w, h, nx, c, time.time() - t, source, whole=tag in ("c2", "c3"))


def c5check(port):
    """The replica against the unmodified reference on C5's first outer iteration (≈6 min of
    the reference on one core): bitwise-identical records and factors."""
    c = CONFIGS["c5"]
    x, w0, h0 = inputs(port, c)
    cfg = preset(c["alg"], max_outer_iterations=1)
    port.threads = os.cpu_count()
    t = time.time()
    a = port.run_dense(x, w0, h0, cfg)
    ta = time.time() - t
    t = time.time()
    b = Oracle("reference").run_dense(x, w0, h0, cfg)
    tb = time.time() - t
    same = all(np.array_equal(a[0][k], b[0][k]) for k in ("error", "beta", "restarted")) and \
        np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) and a[3] == b[3]
    meta_path = os.path.join(OUT, "golden_long.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    meta["c5check"] = dict(iterations=1, bitwise=bool(same), replica_seconds=round(ta, 1),
                           reference_seconds=round(tb, 1), error=b[0]["error"].tolist())
    json.dump(meta, open(meta_path, "w"), indent=1)
    print(f"c5check: bitwise={same} replica {ta:.1f}s reference {tb:.1f}s", flush=True)
    assert same


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4", "c5"])

"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It calls the unmodified reference headers compiled in place
(oracle/_ref/libenmf_ref.so, built by oracle/Makefile from
/root/reference/proj/include) through ref_shim.cpp — not the C restatement —
so the fixtures pin the restatement (tests/test_oracle.py) and the GPU path
(tests/test_gpu_parity.py) to the reference's own outputs.  The GPU box has no
/root/reference; it only reads these committed .npz files.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, default_config, preset  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
PRESETS = ["e-ahals-hp3", "e-ahals-hp1", "e-anls-hp1", "anls", "ahals", "e-anls-hp3"]


def save_run(R, tag, x, w0, h0, cfg, meta):
    rec, w, h, nx = R.run_dense(x, w0, h0, cfg)
    np.savez_compressed(os.path.join(OUT, f"{tag}.npz"), error=rec["error"],
                        relative_error=rec["relative_error"], beta=rec["beta"],
                        restarted=rec["restarted"], w=w, h=h, norm_x=nx)
    meta[tag] = {k: getattr(cfg, k) for k, _ in cfg._fields_}
    meta[tag]["final_relative_error"] = float(rec["relative_error"][-1])
    meta[tag]["restarts"] = int(rec["restarted"].sum())


def csr_fixtures(R, meta):
    """C4-shaped CSR (gen_docs: lognormal document lengths, Zipf term ids, tf·idf, L2 columns)
    at 300×120, r=6, through enmf::run<SparseMatrix> (linalg.hpp:86-146)."""
    gen = Oracle("port")       # data generator only (orc_gen_docs); the runs are the reference's
    off, cidx, vals = gen.gen_docs(300, 120, 4)
    m, n, r = 300, 120, 6
    w0, h0 = R.random_init(m, n, r, 9)
    np.savez_compressed(os.path.join(OUT, "csr_inputs.npz"), off=off, cidx=cidx, vals=vals, w0=w0, h0=h0,
                        m=m, n=n)
    for name in ["e-ahals-hp3", "e-anls-hp1"]:
        cfg = preset(name, max_outer_iterations=40)
        rec, w, h, nx = R.run_csr(off, cidx, vals, m, n, w0, h0, cfg)
        tag = f"csr_{name}"
        np.savez_compressed(os.path.join(OUT, f"{tag}.npz"), error=rec["error"],
                            relative_error=rec["relative_error"], beta=rec["beta"],
                            restarted=rec["restarted"], w=w, h=h, norm_x=nx)
        meta[tag] = {k: getattr(cfg, k) for k, _ in cfg._fields_}
        meta[tag]["final_relative_error"] = float(rec["relative_error"][-1])


def main():
    R = Oracle("reference")
    if len(sys.argv) > 1 and sys.argv[1] == "--csr-only":
        with open(os.path.join(OUT, "golden.json")) as f:
            meta = json.load(f)
        csr_fixtures(R, meta)
        with open(os.path.join(OUT, "golden.json"), "w") as f:
            json.dump(meta, f, indent=1, sort_keys=True, default=float)
        print("wrote CSR fixtures")
        return
    meta = {}
    # Config 1 (BASELINE.json configs[0]): gen_lowrank(200,200,20,seed=1), random_init(...,seed=2), 200 iterations.
    x = R.gen_lowrank(200, 200, 20, 1)
    w0, h0 = R.random_init(200, 200, 20, 2)
    np.savez_compressed(os.path.join(OUT, "c1_inputs.npz"), x=x, w0=w0, h0=h0)
    for name in PRESETS:
        save_run(R, f"c1_{name}", x, w0, h0, preset(name, max_outer_iterations=200), meta)
    # Small variants exercising every SolverConfig branch (hp 1/2/3, literal hp1,
    # momentum off, beta0 = 0, forced sweep count) on a 28×22 r=5 dense X
    # (acceptance.cpp:278-317 uses this shape).
    rng = np.random.default_rng(61)
    xs = rng.random((28, 22))
    ws, hs = R.random_init(28, 22, 5, 600)
    np.savez_compressed(os.path.join(OUT, "small_inputs.npz"), x=xs, w0=ws, h0=hs)
    variants = {
        "hals_hp2": dict(inner_h=1, inner_w=1, hp=2, gamma=1.01, gamma_bar=1.005),
        "hals_hp1_literal": dict(inner_h=1, inner_w=1, hp=1, literal_hp1_order=1, gamma=1.01, gamma_bar=1.005),
        "exact_hp2": dict(hp=2),
        "exact_hp1_literal": dict(hp=1, literal_hp1_order=1),
        "hals_noextrap": dict(inner_h=1, inner_w=1, hp=3, extrapolation_enabled=0),
        "hals_beta0": dict(inner_h=1, inner_w=1, hp=3, beta0=0.0),
        "mixed_hals_exact": dict(inner_h=1, inner_w=0, hp=3, gamma=1.01, gamma_bar=1.005),
        "hals_sweeps3": dict(inner_h=1, inner_w=1, hp=3, inner_max_sweeps=3, gamma=1.01, gamma_bar=1.005),
    }
    for tag, kw in variants.items():
        save_run(R, f"small_{tag}", xs, ws, hs, default_config(max_outer_iterations=40, **kw), meta)
    # Dead starting column: W0 column 2 all zero -> degenerate Gram diagonal ->
    # deterministic reinit (test_engine.cpp:449-465).
    wd = ws.copy()
    wd[:, 2] = 0.0
    np.savez_compressed(os.path.join(OUT, "reinit_inputs.npz"), x=xs, w0=wd, h0=hs)
    save_run(R, "reinit_hals", xs, wd, hs, default_config(max_outer_iterations=20, inner_h=1, inner_w=1, hp=3,
                                                           gamma=1.01, gamma_bar=1.005, reinit_seed=7), meta)
    save_run(R, "reinit_exact", xs, wd, hs, default_config(max_outer_iterations=20, hp=1, reinit_seed=7), meta)
    # Kernel-level fixtures: hals_solve / active_set_solve on a seeded problem.
    g = np.random.default_rng(5)
    wk = g.random((40, 12)); xk = g.random((40, 30))
    G = R.gram(wk); Cm = R.cross_wx(wk, xk)
    h0k = g.random((12, 30)) - 0.3
    hh, _ = R.hals_solve(G, Cm, h0k, 25, 0.01)
    ha, _ = R.active_set_solve(G, Cm, np.abs(h0k))
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), w=wk, x=xk, gram=G, cross=Cm,
                        xht=R.cross_xht(xk, g.random((12, 30))), h0=h0k, hals=hh, bpp=ha)
    csr_fixtures(R, meta)
    # Known answers quoted in SURVEY.md §6.2 for config 1 (hp3 / hp1).
    meta["known_answers"] = {"c1_e-ahals-hp3_final_relative_error": 7.8674950787740083e-4,
                             "c1_e-ahals-hp1_final_relative_error": 1.2721814731209598e-3,
                             "c1_restarts": 5}
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True, default=float)
    print("wrote", len(meta), "fixtures to", OUT)


if __name__ == "__main__":
    main()

"""Engine-level A/B of the sweep kernels (run once per ENMF_HALS_KERNEL value): a C5-like problem
with n = 32768 columns (sweep_tm holds 6-7 tiles per sub-partition on the H side)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1805_06604_b200 as E

m, n, r = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 32768, 128
rng = np.random.default_rng(7)
x = rng.random((m, r)) @ rng.random((r, n)) + np.abs(0.01 * rng.standard_normal((m, n)))
w0, h0 = rng.random((m, r)), rng.random((r, n))
cfg = E.algorithm_config("e-ahals-hp3")
cfg.max_outer_iterations = 8
rec = E.Context(0).run(x, w0, h0, cfg, E.TimingMode.none)
print("inner_h", rec.column("inner_h_count").tolist())
print("inner_w", rec.column("inner_w_count").tolist())
print("error", " ".join(f"{v:.12e}" for v in rec.column("error")))

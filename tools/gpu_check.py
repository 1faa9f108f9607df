"""Quick GPU bring-up check: C1 parity (exact + fast) and a C5 timing probe."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1805_06604_b200 as E
from oracle.oracle import Oracle, preset

P = Oracle("port")
x = P.gen_lowrank(200, 200, 20, 1)
w0, h0 = P.random_init(200, 200, 20, 2)
ctx = E.Context()
for name in ["e-ahals-hp3", "e-ahals-hp1", "e-anls-hp1", "anls", "ahals", "e-anls-hp3"]:
    ref = P.run_dense(x, w0, h0, preset(name, max_outer_iterations=200))
    for prec in [E.Precision.fp64_exact, E.Precision.fp64]:
        cfg = E.algorithm_config(name)
        cfg.max_outer_iterations = 200
        cfg.precision = prec
        t = time.time()
        try:
            rec = ctx.run(x, w0, h0, cfg, E.TimingMode.none)
        except Exception as e:
            print(name, prec.name, "ERROR", type(e).__name__, e); continue
        dt = time.time() - t
        err = rec.column("error"); rs = rec.column("restarted").astype(int)
        re_ = ref[0]["error"]
        n = min(len(err), len(re_))
        dev = np.max(np.abs(err[:n] - re_[:n]) / np.maximum(re_[:n], 1e-300))
        bit = np.array_equal(err, re_) and np.array_equal(rec.factors.w, ref[1]) and np.array_equal(rec.factors.h, ref[2])
        wdev = np.max(np.abs(rec.factors.w - ref[1])) / np.max(np.abs(ref[1]))
        hdev = np.max(np.abs(rec.factors.h - ref[2])) / np.max(np.abs(ref[2]))
        print(f"{name:12s} {prec.name:10s} n={len(err)} bitwise={bit} restarts_eq={np.array_equal(rs, ref[0]['restarted'])} "
              f"maxrel_err_dev={dev:.2e} W={wdev:.2e} H={hdev:.2e} sweeps_eq={np.array_equal(rec.column('inner_h_count'), ref[0]['inner_h'])} t={dt:.3f}s")
        if not bit and prec == E.Precision.fp64_exact:
            k = np.nonzero(err[:n] != re_[:n])[0]
            print("   first mismatch at", k[:5], err[k[:3]] if len(k) else None, re_[k[:3]] if len(k) else None)
            print("   sweeps dev", rec.column('inner_h_count')[:8], ref[0]['inner_h'][:8], rec.column('inner_w_count')[:8], ref[0]['inner_w'][:8])

# C5 probe
import torch
m = n = int(os.environ.get("C5N", "32768")); r = 128
g = torch.Generator(device="cuda").manual_seed(1)
W0 = torch.rand(m, r, device="cuda", dtype=torch.float64, generator=g)
H0 = torch.rand(r, n, device="cuda", dtype=torch.float64, generator=g)
X = W0 @ H0 + 0.01 * torch.randn(m, n, device="cuda", dtype=torch.float64, generator=g).abs()
Wi = torch.rand(m, r, device="cuda", dtype=torch.float64, generator=g)
Hi = torch.rand(r, n, device="cuda", dtype=torch.float64, generator=g)
ctx.load_device(X.data_ptr(), m, n)
cfg = E.algorithm_config("e-ahals-hp3")
for K in [1, 5]:
    cfg.max_outer_iterations = K
    torch.cuda.synchronize(); t = time.time()
    rec = ctx.solve_device(Wi.data_ptr(), Hi.data_ptr(), r, cfg)
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"C5 K={K}: {dt*1e3:.1f} ms total, rel errs {[f'{v:.4e}' for v in rec.column('relative_error')]}, "
          f"sweeps H {list(rec.column('inner_h_count'))} W {list(rec.column('inner_w_count'))}")

"""Where the end-to-end C5 call's time goes: host→device copy, begin() phases
(ENMF_TRACE_BEGIN), iterations, and the copy back — timed on a fresh context twice."""
import os, sys, time
os.environ["ENMF_TRACE_BEGIN"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1805_06604_b200 as E

M = N = 32768
R = 128
g = torch.Generator(device="cuda").manual_seed(1)
x = (torch.rand(M, R, dtype=torch.float64, device="cuda", generator=g) @
     torch.rand(R, N, dtype=torch.float64, device="cuda", generator=g))
x += (0.01 * torch.randn(M, N, dtype=torch.float64, device="cuda", generator=g)).abs_()
xh = torch.empty(x.shape, dtype=torch.float64, pin_memory=True)
xh.copy_(x)
del x
torch.cuda.empty_cache()
rng = np.random.default_rng(2)
w0, h0 = rng.random((M, R)), rng.random((R, N))
# raw pinned H2D bandwidth on this box
d = torch.empty((M, N), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(xh, non_blocking=True); torch.cuda.synchronize()
print(f"pinned H2D of X: {(time.perf_counter() - t) * 1e3:.1f} ms = {M * N * 8 / (time.perf_counter() - t) / 1e9:.1f} GB/s",
      file=sys.stderr)
del d
torch.cuda.empty_cache()
xn = xh.numpy()
for rep in range(2):
    cfg = E.algorithm_config("e-ahals-hp3")
    cfg.max_outer_iterations = 20
    ctx = E.Context(0)
    t = time.perf_counter()
    rec = ctx.run(xn, w0, h0, cfg, E.TimingMode.none)
    print(f"rep {rep}: run_dense {time.perf_counter() - t:.3f} s", file=sys.stderr)
    ctx.close()

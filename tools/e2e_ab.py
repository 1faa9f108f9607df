"""End-to-end C5 call (enmf_gpu_run_dense on pinned host buffers, fresh context per call) with the
X upload overlapped with begin() (default) or completed first (ENMF_X_UPLOAD=sync): run once per mode."""
import os, sys, time
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
pin = lambda a: torch.empty(a.shape, dtype=torch.float64, pin_memory=True).copy_(torch.from_numpy(a))
w0, h0 = pin(rng.random((M, R))).numpy(), pin(rng.random((R, N))).numpy()
xn = xh.numpy()
for rep in range(4):
    cfg = E.algorithm_config("e-ahals-hp3")
    cfg.max_outer_iterations = 20
    ctx = E.Context(0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    rec = ctx.run(xn, w0, h0, cfg, E.TimingMode.none)
    print(f"mode {os.environ.get('ENMF_X_UPLOAD', 'overlap')} rep {rep}: run_dense {time.perf_counter() - t:.3f} s", file=sys.stderr, flush=True)
    ctx.close()

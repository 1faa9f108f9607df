"""Phases of one C5 run through the C-ABI: upload, begin (X digit cuts, e(0)), iterations."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_06604_b200 as E
import bench
dev = torch.device("cuda", 0)
w0, h0, wi, hi = bench.gen_factors(dev, 1234)
x = bench.gen_block(w0, h0, 0, bench.M, 0, bench.N, 1234)
xh = torch.empty(x.shape, dtype=torch.float64, pin_memory=True).copy_(x)
wh = torch.empty(wi.shape, dtype=torch.float64, pin_memory=True).copy_(wi)
hh = torch.empty(hi.shape, dtype=torch.float64, pin_memory=True).copy_(hi)
del x
torch.cuda.empty_cache()
cfg = bench.cfg_c5(5)
for rep in range(2):
    ctx = E.Context(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ctx.load(xh.numpy()); torch.cuda.synchronize()
    t1 = time.perf_counter(); ctx.begin(wh.numpy(), hh.numpy(), cfg); ctx.sync(); torch.cuda.synchronize()
    t2 = time.perf_counter(); ctx.step(5); ctx.sync()
    t3 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.1f} ms  begin {1e3*(t2-t1):.1f} ms  5 iterations {1e3*(t3-t2):.1f} ms", flush=True)
    ctx.end(); ctx.close()

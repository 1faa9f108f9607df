"""Relative error / bias of TF32 tensor-core products (cuBLAS, FP32 accumulation) on C5-like data."""
import torch
torch.manual_seed(0)
dev = "cuda"
m = n = 32768; r = 128
w0 = torch.rand(m, r, device=dev, dtype=torch.float64)
h0 = torch.rand(r, n, device=dev, dtype=torch.float64)
x = (w0 @ h0[:, :4096]).add_(torch.randn(m, 4096, device=dev, dtype=torch.float64).abs_().mul_(0.01))
wt = torch.rand(r, m, device=dev, dtype=torch.float64)
ref = wt @ x
for tf in (True, False):
    torch.backends.cuda.matmul.allow_tf32 = tf
    c = (wt.float() @ x.float()).double()
    rel = (c - ref) / ref
    print(f"allow_tf32={tf}: mean rel {rel.mean().item():.3e}  rms rel {rel.pow(2).mean().sqrt().item():.3e}  "
          f"max {rel.abs().max().item():.3e}")
# K-split accumulation in FP32 vs FP64
torch.backends.cuda.matmul.allow_tf32 = True
acc = torch.zeros_like(ref)
for k0 in range(0, m, 1024):
    acc += (wt[:, k0:k0+1024].float() @ x[k0:k0+1024].float()).double()
rel = (acc - ref) / ref
print(f"tf32, FP64 sum of 1024-wide K chunks: mean rel {rel.mean().item():.3e} rms {rel.pow(2).mean().sqrt().item():.3e}")

"""INT8 tensor-core throughput on this B200 through cuBLASLt (torch._int_mm),
for the Ozaki-split cross products: M (stacked factor slices) × K=32768 × N=32768."""
import torch
torch.backends.cuda.matmul.allow_tf32 = True
dev = "cuda"
K = N = 32768
for M in (128, 256, 512, 768, 1024):
    a = torch.randint(-127, 127, (M, K), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 127, (K, N), dtype=torch.int8, device=dev)
    for layout in ("b_rowmajor", "b_colmajor"):
        bb = b if layout == "b_rowmajor" else b.t().contiguous().t()
        try:
            c = torch._int_mm(a, bb)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                c = torch._int_mm(a, bb)
            e1.record(); e1.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"int8 M={M} {layout}: {ms:.3f} ms  {2*M*K*N/ms/1e9:.0f} TOPS", flush=True)
        except Exception as ex:
            print(f"int8 M={M} {layout}: {type(ex).__name__}: {str(ex)[:120]}", flush=True)
# TF32 for reference
a = torch.rand(128, K, device=dev); b = torch.rand(K, N, device=dev)
c = a @ b; torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): c = a @ b
e1.record(); e1.synchronize(); ms = e0.elapsed_time(e1) / 5
print(f"tf32 M=128: {ms:.3f} ms {2*128*K*N/ms/1e9:.0f} TFLOPS")

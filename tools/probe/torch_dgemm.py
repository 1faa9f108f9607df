import torch, time
def bench(M,N,K,dt=torch.float64, transA=False, transB=False, it=10):
    a = torch.rand(K,M,device='cuda',dtype=dt).t() if transA else torch.rand(M,K,device='cuda',dtype=dt)
    b = torch.rand(N,K,device='cuda',dtype=dt).t() if transB else torch.rand(K,N,device='cuda',dtype=dt)
    for _ in range(2): c = a@b
    torch.cuda.synchronize()
    best=1e9
    for _ in range(it):
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); c=a@b; e.record(); torch.cuda.synchronize(); best=min(best,s.elapsed_time(e))
    print(f"{dt} M={M} N={N} K={K} tA={transA} tB={transB}: {best:.3f} ms  {2*M*N*K/best/1e9:.2f} TFLOP/s")
bench(8192,8192,8192)
# C5 shapes: WᵀX : (128 x 32768)(32768 x 32768), A = W^T given W m x r row-major
bench(128,32768,32768, transA=True)
# X Hᵀ : (32768x32768)(32768x128), B = H^T with H r x n row-major
bench(32768,128,32768, transB=True)
bench(8192,8192,8192, dt=torch.float32)
torch.backends.cuda.matmul.allow_tf32=True
bench(8192,8192,8192, dt=torch.float32)
bench(128,32768,32768, dt=torch.float32, transA=True)

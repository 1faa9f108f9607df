"""Pinned host->device bandwidth of X (8.6 GB) on 1, 2, 4, 8 streams and in chunks on one stream (55.6 GB/s every way:
the X upload of the end-to-end call cannot be sped up by splitting it).
"""
import torch, time
n = 32768 * 32768
x = torch.empty(n, dtype=torch.float64, pin_memory=True)
x.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        t = time.perf_counter()
        ch = n // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * ch:(i + 1) * ch].copy_(x[i * ch:(i + 1) * ch], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"{k} streams: {best*1e3:.1f} ms = {n*8/best/1e9:.1f} GB/s")
# chunked on one stream
for nch in (8, 32):
    torch.cuda.synchronize(); t = time.perf_counter()
    ch = n // nch
    for i in range(nch):
        d[i*ch:(i+1)*ch].copy_(x[i*ch:(i+1)*ch], non_blocking=True)
    torch.cuda.synchronize(); print(f"1 stream {nch} chunks: {(time.perf_counter()-t)*1e3:.1f} ms")

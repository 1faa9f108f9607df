// Does scalar FP64 on one SM sub-partition (SMSP) slow down while the OTHER three SMSPs
// stream DMMA?  (Same-SMSP contention is in contend_probe.cu / pipe_probe.cu.)
// Warp w runs on SMSP w % 4.  Modes:
//   flood  = number of DMMA-streaming warps per SMSP on SMSPs 0..2 (0, 1, 2)
//   scalar = what warp 3 (SMSP 3) does: 0 dependent DFMA chain, 1 independent DFMAs (8 chains),
//            2 an 8-row triangular HALS-like chain over 3 columns per lane
// Reports cycles per scalar op on SMSP 3 and cycles per DMMA per SMSP on SMSPs 0..2.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void k(long long* out, double* sink, int iters, int flood, int scalar, int same) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int smsp = warp & 3;
  const int scal_warp = same ? 0 : 3;
  if (warp == scal_warp) {
    long long t0 = clock64();
    double x = lane * 1e-3 + 1.0, y = 1.0000001;
    if (scalar == 0) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x = fma(x, y, 1e-9);
      }
      sink[threadIdx.x] = x;
    } else if (scalar == 1) {
      double c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = x + j;
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) c[j] = fma(c[j], y, 1e-9);
      }
      double s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) s += c[j];
      sink[threadIdx.x] = s;
    } else {
      // 8-row block solve for 3 columns per lane (the shape of a row warp serving 3 groups)
      double g[28], inv[8], bb[3][8], gain = 0;
#pragma unroll
      for (int j = 0; j < 28; ++j) g[j] = 1e-3 * (j + 1);
#pragma unroll
      for (int j = 0; j < 8; ++j) inv[j] = 0.9 + 0.01 * j;
      for (int it = 0; it < iters / 8; ++it) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int j = 0; j < 8; ++j) bb[c][j] = x + c + j * 0.1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double t = bb[c][i] * inv[i];
            const double h = t > 0.0 ? t : 0.0;
#pragma unroll
            for (int l = i + 1; l < 8; ++l) bb[c][l] = fma(-g[l * (l - 1) / 2 + i], h, bb[c][l]);
            gain = fma(t - h, t + h, gain);
          }
        }
        x = gain * 1e-30 + 1.0;
      }
      sink[threadIdx.x] = gain;
    }
    long long t1 = clock64();
    if (lane == 0) out[0] = t1 - t0;
  } else if (smsp != scal_warp % 4 || same) {
    // DMMA flooders: `flood` warps on each of SMSPs 0..2 (or on SMSP 0 for `same`)
    const int idx = warp / 4;                   // 0.. per SMSP
    const bool on = same ? (smsp == 0 && idx >= 1 && idx <= flood) : (smsp < 3 && idx < flood);
    if (!on) return;
    double c[4][2] = {};
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    long long t0 = clock64();
    for (int it = 0; it < iters * 4; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    long long t1 = clock64();
    sink[threadIdx.x] = c[0][0] + c[1][1] + c[2][0] + c[3][1];
    if (lane == 0 && idx == (same ? 1 : 0) && smsp == 0) out[1] = t1 - t0;
  }
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 16);
  cudaMalloc(&s, 1024 * 8);
  const int it = 4000;
  const char* names[3] = {"dependent DFMA chain", "8 independent DFMA chains", "8-row block solve x3 cols"};
  for (int same = 0; same < 2; ++same)
    for (int sc = 0; sc < 3; ++sc)
      for (int fl = 0; fl <= 2; ++fl) {
        cudaMemset(d, 0, 16);
        k<<<1, 384>>>(d, s, 16, fl, sc, same);
        k<<<1, 384>>>(d, s, it, fl, sc, same);
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const double ops = sc == 0 ? it * 16.0 : sc == 1 ? it * 16.0 : (it / 8) * 8.0;   // per op / per row
        printf("%s  scalar: %-28s flood %d warps/SMSP: %8.1f cycles per %s;  DMMA warp %.1f cycles/DMMA\n",
               same ? "SAME SMSP " : "OTHER SMSP", names[sc], fl, (double)h[0] / ops, sc == 2 ? "row (3 cols)" : "op",
               fl ? (double)h[1] / (it * 16.0) : 0.0);
      }
  return 0;
}

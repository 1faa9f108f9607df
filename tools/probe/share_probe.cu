// How is the FP64 pipe of ONE SM sub-partition shared between a DMMA-streaming warp and S scalar
// FP64 warps (S = 1..4)?  Warps 0, 4, 8, ... run on SMSP 0; warp 0 streams DMMA.8x8x4, warps
// 4, 8, .. run scalar FP64 (mode 0: one dependent DFMA chain, 1: 8 independent chains, 2: an
// 8-row HALS block solve with gains, one column per lane, 3: the same with two columns per lane).
// Reports cycles per scalar op (or per block) of the slowest scalar warp and cycles per DMMA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NC>
__device__ double block_solve(double x, int iters) {
  double g[28], inv[8], gk[8], bb[NC][8], xo[NC][8], gain = 0;
#pragma unroll
  for (int j = 0; j < 28; ++j) g[j] = 1e-3 * (j + 1);
#pragma unroll
  for (int j = 0; j < 8; ++j) { inv[j] = 0.9 + 0.01 * j; gk[j] = 0.5 + 0.01 * j; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int j = 0; j < 8; ++j) { bb[c][j] = (x + c + j * 0.1 - 0.3) * inv[j]; xo[c][j] = x * 0.5 + j; }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double t = bb[c][i];
        const double h = t > 0.0 ? t : 0.0;
#pragma unroll
        for (int l = i + 1; l < 8; ++l) bb[c][l] = fma(-g[l * (l - 1) / 2 + i], h, bb[c][l]);
        const double u = xo[c][i] - h, v = xo[c][i] + h;
        gain = fma(u * gk[i], fma(-2.0, t, v), gain);
      }
    }
    x = gain * 1e-30 + 1.0;
  }
  return gain;
}

__global__ void k(long long* out, double* sink, int iters, int nscal, int mode, int flood) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp & 3) return;
  const int idx = warp >> 2;
  if (idx == 0) {
    if (!flood) return;
    double c[8][2] = {};
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    long long t0 = clock64();
    for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    long long t1 = clock64();
    sink[threadIdx.x] = c[0][0] + c[1][1] + c[2][0] + c[3][1] + c[4][0] + c[5][0] + c[6][0] + c[7][0];
    if (lane == 0) out[0] = t1 - t0;
    return;
  }
  if (idx > nscal) return;
  long long t0 = clock64();
  double x = lane * 1e-3 + 1.0, y = 1.0000001, res;
  if (mode == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x = fma(x, y, 1e-9);
    }
    res = x;
  } else if (mode == 1) {
    double c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = x + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = fma(c[j], y, 1e-9);
    }
    res = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) res += c[j];
  } else if (mode == 2) {
    res = block_solve<1>(x, iters / 4);
  } else {
    res = block_solve<2>(x, iters / 4);
  }
  long long t1 = clock64();
  sink[threadIdx.x] = res;
  if (lane == 0) out[idx] = t1 - t0;
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 64);
  cudaMalloc(&s, 1024 * 8);
  const int it = 4000;
  const char* names[4] = {"dependent DFMA chain", "8 independent DFMA chains", "block solve+gains, 1 col/lane",
                          "block solve+gains, 2 col/lane"};
  for (int mode = 0; mode < 4; ++mode)
    for (int fl = 0; fl < 2; ++fl)
      for (int ns = 1; ns <= 4; ++ns) {
        cudaMemset(d, 0, 64);
        k<<<1, 32 * 4 * 5>>>(d, s, 16, ns, mode, fl);
        cudaMemset(d, 0, 64);
        k<<<1, 32 * 4 * 5>>>(d, s, it, ns, mode, fl);
        long long h[8];
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 1; i <= ns; ++i) mx = h[i] > mx ? h[i] : mx;
        const double ops = mode < 2 ? it * 16.0 : it / 4.0;
        printf("%-30s DMMA flood %d, %d scalar warps: %8.1f cycles per %s per warp;  DMMA %.1f cycles\n", names[mode],
               fl, ns, (double)mx / ops, mode < 2 ? "op" : "block", fl ? (double)h[0] / (it * 64.0) : 0.0);
      }
  return 0;
}

// Does FP64 scalar work (DADD chains) contend with DMMA on the same SM sub-partition?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(long long* out, double* sink, int iters, int flood_warps, int chain_kind) {
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    double x = threadIdx.x * 1e-3, y = 1.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (chain_kind == 0) x = x + y;          // DADD chain
        else x = x * 1.0000001;                  // DMUL chain
      }
    }
    long long t1 = clock64();
    sink[threadIdx.x] = x;
    if (threadIdx.x == 0) out[0] = t1 - t0;
  } else if ((warp % 4) == 0 && warp / 4 <= flood_warps) {
    double c[4][2] = {};
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    for (int it = 0; it < iters * 4; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    sink[threadIdx.x] = c[0][0] + c[1][1] + c[2][0] + c[3][1];
  }
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 8); cudaMalloc(&s, 4096 * 8);
  long long h; int it = 2000;
  for (int kind = 0; kind < 2; ++kind)
    for (int fw = 0; fw <= 3; ++fw) {
      k<<<1, 32 * (1 + 4 * fw)>>>(d, s, 10, fw, kind);
      k<<<1, 32 * (1 + 4 * fw)>>>(d, s, it, fw, kind);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%s chain with %d DMMA-flooding warps on the same SMSP: %.1f cycles/op\n", kind ? "DMUL" : "DADD", fw,
             (double)h / (it * 16));
    }
  return 0;
}

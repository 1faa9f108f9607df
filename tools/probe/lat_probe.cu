// Latency probe on sm_100a: dependent DMMA chains (1..8 chains/warp), DFMA, SHFL.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k_dmma(long long* out, double* sink, int iters) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  sink[threadIdx.x] = s;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void k_dfma(long long* out, double* sink, int iters) {
  double x = threadIdx.x, a = 1.0000001, b = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x = fma(x, a, b);
  }
  long long t1 = clock64();
  sink[threadIdx.x] = x;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void k_shfl(long long* out, double* sink, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1.0;
  }
  long long t1 = clock64();
  sink[threadIdx.x] = x;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void k_lds(long long* out, double* sink, int iters) {
  __shared__ int idx[64];
  if (threadIdx.x < 64) idx[threadIdx.x] = (threadIdx.x + 1) & 31;
  __syncthreads();
  int p = threadIdx.x & 31;
  long long t0 = clock64();
  for (int it = 0; it < iters * 8; ++it) p = idx[p];
  long long t1 = clock64();
  sink[threadIdx.x] = p;
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 8); cudaMalloc(&s, 4096 * 8);
  long long h; int it = 1000;
#define RUN(K, name, per) K<<<1, 32>>>(d, s, 10); K<<<1, 32>>>(d, s, it); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("%-22s %.1f cycles per op\n", name, (double)h / (it * (per)));
  RUN(k_dmma<1>, "DMMA 1 chain", 1);
  RUN(k_dmma<2>, "DMMA 2 chains (/dmma)", 2);
  RUN(k_dmma<4>, "DMMA 4 chains (/dmma)", 4);
  RUN(k_dmma<8>, "DMMA 8 chains (/dmma)", 8);
  RUN(k_dmma<16>, "DMMA 16 chains (/dmma)", 16);
  RUN(k_dfma, "DFMA dependent", 8);
  RUN(k_shfl, "SHFL(double)+DADD dep", 8);
  RUN(k_lds, "LDS dependent", 8);
  // 4 warps on one SM, 8 chains each: per-SMSP throughput
  k_dmma<8><<<1, 128>>>(d, s, it); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %.1f cycles per dmma per warp\n", "DMMA 4 warps x 8ch", (double)h / (it * 8));
  k_dmma<8><<<1, 256>>>(d, s, it); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %.1f cycles per dmma per warp\n", "DMMA 8 warps x 8ch", (double)h / (it * 8));
  return 0;
}

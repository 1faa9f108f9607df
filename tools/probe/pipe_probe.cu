// Cost of scalar FP64 instructions issued next to a DMMA stream on the same SM
// sub-partition: warp 0 floods DMMA.8x8x4 (4 independent accumulators), warp 4
// (same SMSP) issues NS scalar DFMAs in bursts of B independent ops.  Prints the
// DMMA warp's cycles per DMMA and the extra DMMA-pipe cycles per scalar op.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int B>
__global__ void k(long long* out, double* sink, int nd, int ns, int swap) {
  const int warp = (threadIdx.x >> 5) ^ (swap ? 4 : 0);   // swap: scalar warp is the older one
  if (warp == 0) {
    double c[4][2] = {};
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    long long t0 = clock64();
    for (int it = 0; it < nd / 4; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    sink[threadIdx.x] = c[0][0] + c[1][1] + c[2][0] + c[3][1];
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[0] = t1 - t0;
  } else if (warp == 4 && ns > 0) {
    double x[B];
#pragma unroll
    for (int i = 0; i < B; ++i) x[i] = threadIdx.x * 1e-3 + i;
    const double y = 1.0000001, z = 1e-9;
    long long t0 = clock64();
    for (int it = 0; it < ns / B; ++it) {
#pragma unroll
      for (int i = 0; i < B; ++i) x[i] = fma(x[i], y, z);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < B; ++i) s += x[i];
    long long t1 = clock64();
    sink[threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) out[1] = t1 - t0;
  }
}
template <int B>
void run(long long* d, double* s, int nd, int ns, int swap = 0) {
  long long h[2] = {0, 0};
  k<B><<<1, 160>>>(d, s, 64, ns ? 64 : 0, swap);
  cudaMemset(d, 0, 16);
  k<B><<<1, 160>>>(d, s, nd, ns, swap);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%s burst %2d  scalar ops %6d : DMMA warp %.2f cycles/DMMA (%lld cyc), scalar warp %lld cyc (%.1f/op)\n",
         swap ? "scalar=warp0" : "dmma=warp0  ", B, ns, (double)h[0] / nd, h[0], h[1], ns ? (double)h[1] / ns : 0.0);
}
int main() {
  long long* d; double* s; cudaMalloc(&d, 16); cudaMalloc(&s, 4096 * 8);
  const int nd = 8192;
  run<1>(d, s, nd, 0);
  for (int ns : {256, 1024}) {
    run<1>(d, s, nd, ns);
    run<2>(d, s, nd, ns);
    run<4>(d, s, nd, ns);
    run<8>(d, s, nd, ns);
    run<16>(d, s, nd, ns);
    run<1>(d, s, nd, ns, 1);
    run<2>(d, s, nd, ns, 1);
    run<4>(d, s, nd, ns, 1);
    run<8>(d, s, nd, ns, 1);
  }
  return 0;
}

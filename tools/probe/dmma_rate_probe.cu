// What sets the DMMA.8x8x4 issue rate of ONE warp per SM sub-partition: the number of independent
// accumulators (ACC), and whether consecutive DMMAs share their A / B operand registers.
//   mode 0: same A, same B for every DMMA (the peak probe's pattern)
//   mode 1: same A for a run of ACC DMMAs, B differs per DMMA (the sweep's product loop)
//   mode 2: A and B differ per DMMA
// Reports cycles per DMMA (clock64 of warp 0).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b) : "memory");
}

template <int ACC, int MODE>
__global__ void k(long long* out, double* sink, int iters) {
  double c[ACC][2], a[ACC], b[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) {
    c[i][0] = c[i][1] = 0.0;
    a[i] = 1.0 + 1e-3 * (threadIdx.x + i);
    b[i] = 0.999 - 1e-3 * (threadIdx.x + 2 * i);
  }
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 2; ++rep)
#pragma unroll
      for (int i = 0; i < ACC; ++i)
        dmma(c[i][0], c[i][1], MODE == 2 ? a[i] : a[rep], MODE == 0 ? b[0] : b[i]);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

template <int ACC, int MODE>
void run(long long* d, double* s, const char* what) {
  const int it = 4000;
  k<ACC, MODE><<<148, 128>>>(d, s, 16);
  k<ACC, MODE><<<148, 128>>>(d, s, it);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%2d accumulators, %-34s %6.2f cycles per DMMA\n", ACC, what, (double)h / (2.0 * ACC * it));
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 148 * 128 * 8);
  run<4, 0>(d, s, "same A, same B:");
  run<8, 0>(d, s, "same A, same B:");
  run<14, 0>(d, s, "same A, same B:");
  run<4, 1>(d, s, "A per run, B per DMMA:");
  run<8, 1>(d, s, "A per run, B per DMMA:");
  run<14, 1>(d, s, "A per run, B per DMMA:");
  run<16, 1>(d, s, "A per run, B per DMMA:");
  run<4, 2>(d, s, "A and B per DMMA:");
  run<8, 2>(d, s, "A and B per DMMA:");
  run<14, 2>(d, s, "A and B per DMMA:");
  return 0;
}

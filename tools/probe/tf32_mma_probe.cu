// Throughput of the legacy warp-level TF32 MMA (mma.sync.m16n8k8.row.col.f32.tf32.tf32.f32) on
// B200, one warp per SM sub-partition, 4 independent accumulators; vs DMMA.8x8x4 (FP64).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128, 1) k(float* sink, long long* out, int reps) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  float c[4][4] = {};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  long long t1 = clock64();
  float z = 0;
  for (int j = 0; j < 4; ++j) z += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  sink[blockIdx.x * 128 + threadIdx.x] = z;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}
int main() {
  float* s; long long* d; cudaMalloc(&s, 148 * 128 * 4); cudaMalloc(&d, 8);
  const int reps = 4096;
  k<<<148, 128>>>(s, d, 16);
  k<<<148, 128>>>(s, d, reps);
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)h / (reps * 4);
  printf("mma.sync m16n8k8 tf32: %.2f cycles per MMA per warp (1 warp/SMSP) = %.0f FMA/cycle/SMSP -> %.0f TFLOP/s on 148 SMs at 1.965 GHz\n",
         cyc, 1024 / cyc, 1024 / cyc * 2 * 4 * 148 * 1.965e9 / 1e12);
  return 0;
}

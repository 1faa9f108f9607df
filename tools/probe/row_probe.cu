// Cost of the HALS row pass (one 8-row block, one column per lane) of hals::sweep_ws run
// alone by one warp per SM sub-partition: data in shared memory, no barriers.
// Prints cycles per block for variants of the arithmetic.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double pos_part(double t) {
  const long long b = __double_as_longlong(t);
  return (b > 0 && b <= 0x7FF0000000000000LL) ? t : 0.0;
}
template <int V>
__global__ void __launch_bounds__(128, 1) k(const double* gsrc, long long* out, double* sink, int reps) {
  __shared__ double Ss[4][8 * 40];
  __shared__ double Hs[4][16 * 32];
  __shared__ double Gc[48 * 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 8 * 40; i += 32) Ss[warp][i] = 0.1 + 1e-3 * i;
  for (int i = lane; i < 16 * 32; i += 32) Hs[warp][i] = 0.2 + 1e-3 * i;
  for (int i = threadIdx.x; i < 96; i += 128) Gc[i] = (i % 48) >= 28 ? 1.0 + 1e-3 * i : 1e-3 * i;
  __syncthreads();
  double gain = 0.0;
  double cn[8];
  for (int i = 0; i < 8; ++i) cn[i] = 1.0 + i;
  int hoff[4] = {0, 1, 2, 3};
  const long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    double* hrow = Hs[warp] + (rep & 1) * 8 * 32 + lane;
    const double* gc = (V >= 4) ? Gc : Gc + (rep & 1) * 48;
    double bb[8], x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      bb[i] = (V == 1) ? Ss[warp][i * 40 + lane] : __dsub_rn(cn[i], Ss[warp][i * 40 + lane]);
      x[i] = hrow[i * 32 + hoff[i & 3]];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double t = __dmul_rn(bb[i], gc[36 + i]);
      const double h = (V == 5) ? t : (V == 6 ? fmax(t, 0.0) : pos_part(t));
#pragma unroll
      for (int l = i + 1; l < 8; ++l) bb[l] = fma(-gc[l * (l - 1) / 2 + i], h, bb[l]);
      hrow[i * 32 + hoff[i & 3]] = h;
      if (V == 0 || V == 1 || V >= 4) {
        const double u = __dsub_rn(x[i], h), v = __dadd_rn(x[i], h);
        gain = fma(u, fma(gc[28 + i], v, -bb[i]), gain);
      } else if (V == 3) {
        gain = fma(__dsub_rn(x[i], h), gc[28 + i], gain);
      }
    }
    __syncwarp();
  }
  const long long t1 = clock64();
  sink[blockIdx.x * 128 + threadIdx.x] = gain;
  if (lane == 0 && blockIdx.x == 0 && warp == 0) out[0] = t1 - t0;
}
template <int V>
void run(const char* name, long long* d, double* s) {
  const int reps = 4096;
  k<V><<<1, 128>>>(nullptr, d, s, 16);
  k<V><<<1, 128>>>(nullptr, d, s, reps);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-48s %.1f cycles per 8-row block\n", name, (double)h / reps);
}
int main() {
  long long* d; double* s;
  cudaMalloc(&d, 64); cudaMalloc(&s, 148 * 128 * 8);
  run<0>("current (C - S, chain, 4-op gain)", d, s);
  run<1>("C folded into S (no DSUB)", d, s);
  run<2>("no gain", d, s);
  run<3>("2-op gain", d, s);
  run<4>("current, Gram constants loop-invariant", d, s);
  run<5>("same, no max(t, 0)", d, s);
  run<6>("same, fmax(t, 0) (DMNMX)", d, s);
  return 0;
}

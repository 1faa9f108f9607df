// Issue rate of the HALS sweep's block product ("head") on one warp per SM
// sub-partition: 4 accumulators (column tiles), A fragments in registers, B
// fragments from shared memory (LDS.128, swizzled), optional rolling LDG of the
// next A fragments.  Prints cycles per DMMA for each variant.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
constexpr int KS = 32;
template <int V>
__global__ void __launch_bounds__(128, 1) k(const double2* gf, long long* out, double* sink, int reps) {
  extern __shared__ __align__(16) double Hsm[];
  double (*Hs)[128 * 32] = reinterpret_cast<double (*)[128 * 32]>(Hsm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, gt = lane & 3;
  for (int i = lane; i < 128 * 32; i += 32) Hs[warp][i] = 1.0 + 1e-6 * i;
  __syncwarp();
  const int swz = ((gt & 1) << 2) | (gt >> 1);
  const int bx0 = 2 * ((2 * gi) ^ swz), bx1 = 2 * ((2 * gi + 1) ^ swz);
  const double* hs = Hs[warp];
  double A[KS];
  for (int s = 0; s < KS; ++s) A[s] = 1.0 + s * 1e-3 + lane * 1e-5;
  double acc[4][2] = {};
  const double2* g = gf + lane;
  long long t0 = clock64();
  if (V >= 3 && V <= 5) {
    constexpr int D = (V >= 3 && V <= 5) ? V - 2 : 1;   // prefetch distance in k-step pairs
    double2 buf[D + 1][4];
    auto ld = [&](int s, double2 (&b)[4]) {
      const int k0 = 4 * s + gt, k1 = k0 + 4;
      b[0] = *reinterpret_cast<const double2*>(hs + k0 * 32 + bx0);
      b[1] = *reinterpret_cast<const double2*>(hs + k0 * 32 + bx1);
      b[2] = *reinterpret_cast<const double2*>(hs + k1 * 32 + bx0);
      b[3] = *reinterpret_cast<const double2*>(hs + k1 * 32 + bx1);
    };
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int j = 0; j < D; ++j) ld(2 * j, buf[j]);
#pragma unroll
      for (int s = 0; s < KS; s += 2) {
        const int j = s / 2;
        if (j + D < KS / 2) ld(2 * (j + D), buf[(j + D) % (D + 1)]);
        double2 (&b)[4] = buf[j % (D + 1)];
        dmma(acc[0][0], acc[0][1], A[s], b[0].x);
        dmma(acc[1][0], acc[1][1], A[s], b[0].y);
        dmma(acc[2][0], acc[2][1], A[s], b[1].x);
        dmma(acc[3][0], acc[3][1], A[s], b[1].y);
        dmma(acc[0][0], acc[0][1], A[s + 1], b[2].x);
        dmma(acc[1][0], acc[1][1], A[s + 1], b[2].y);
        dmma(acc[2][0], acc[2][1], A[s + 1], b[3].x);
        dmma(acc[3][0], acc[3][1], A[s + 1], b[3].y);
      }
    }
  } else if (V == 9) {   // joint head: one B load feeds two A fragment sets (8 accumulators)
    double acc1[4][2] = {};
    double A1[KS];
    for (int q = 0; q < KS; ++q) A1[q] = 2.0 + q * 1e-3 + lane * 1e-5;
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int s = 0; s < KS; s += 2) {
        const int k0 = 4 * s + gt, k1 = k0 + 4;
        const double2 p0 = *reinterpret_cast<const double2*>(hs + k0 * 32 + bx0);
        const double2 p1 = *reinterpret_cast<const double2*>(hs + k0 * 32 + bx1);
        const double2 q0 = *reinterpret_cast<const double2*>(hs + k1 * 32 + bx0);
        const double2 q1 = *reinterpret_cast<const double2*>(hs + k1 * 32 + bx1);
        dmma(acc[0][0], acc[0][1], A[s], p0.x);
        dmma(acc[1][0], acc[1][1], A[s], p0.y);
        dmma(acc[2][0], acc[2][1], A[s], p1.x);
        dmma(acc[3][0], acc[3][1], A[s], p1.y);
        dmma(acc[0][0], acc[0][1], A[s + 1], q0.x);
        dmma(acc[1][0], acc[1][1], A[s + 1], q0.y);
        dmma(acc[2][0], acc[2][1], A[s + 1], q1.x);
        dmma(acc[3][0], acc[3][1], A[s + 1], q1.y);
        dmma(acc1[0][0], acc1[0][1], A1[s], p0.x);
        dmma(acc1[1][0], acc1[1][1], A1[s], p0.y);
        dmma(acc1[2][0], acc1[2][1], A1[s], p1.x);
        dmma(acc1[3][0], acc1[3][1], A1[s], p1.y);
        dmma(acc1[0][0], acc1[0][1], A1[s + 1], q0.x);
        dmma(acc1[1][0], acc1[1][1], A1[s + 1], q0.y);
        dmma(acc1[2][0], acc1[2][1], A1[s + 1], q1.x);
        dmma(acc1[3][0], acc1[3][1], A1[s + 1], q1.y);
      }
    }
    for (int t = 0; t < 4; ++t) acc[t][0] += acc1[t][0] + acc1[t][1];
  } else
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int s = 0; s < KS; s += 2) {
      const int k0 = 4 * s + gt, k1 = k0 + 4;
      double2 p0, p1, q0, q1;
      if (V == 2) {
        p0 = make_double2(A[s], A[s + 1]); p1 = p0; q0 = p0; q1 = p0;
      } else {
        p0 = *reinterpret_cast<const double2*>(hs + k0 * 32 + bx0);
        p1 = *reinterpret_cast<const double2*>(hs + k0 * 32 + bx1);
        q0 = *reinterpret_cast<const double2*>(hs + k1 * 32 + bx0);
        q1 = *reinterpret_cast<const double2*>(hs + k1 * 32 + bx1);
      }
      dmma(acc[0][0], acc[0][1], A[s], p0.x);
      dmma(acc[1][0], acc[1][1], A[s], p0.y);
      dmma(acc[2][0], acc[2][1], A[s], p1.x);
      dmma(acc[3][0], acc[3][1], A[s], p1.y);
      dmma(acc[0][0], acc[0][1], A[s + 1], q0.x);
      dmma(acc[1][0], acc[1][1], A[s + 1], q0.y);
      dmma(acc[2][0], acc[2][1], A[s + 1], q1.x);
      dmma(acc[3][0], acc[3][1], A[s + 1], q1.y);
      if (V == 1) {
        const double2 n = g[((rep & 15) * 16 + s / 2) * 32];
        A[s] = n.x;
        A[s + 1] = n.y;
      }
    }
  }
  long long t1 = clock64();
  double z = 0;
  for (int t = 0; t < 4; ++t) z += acc[t][0] + acc[t][1];
  sink[blockIdx.x * 128 + threadIdx.x] = z;
  if (lane == 0 && blockIdx.x == 0) out[warp] = t1 - t0;
}
template <int V>
void run(const char* name, double2* gf, long long* d, double* s, int blocks) {
  const int reps = 512;
  cudaFuncSetAttribute((const void*)k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 128 * 32 * 8);
  k<V><<<blocks, 128, 4 * 128 * 32 * 8>>>(gf, d, s, 8);
  k<V><<<blocks, 128, 4 * 128 * 32 * 8>>>(gf, d, s, reps);
  long long h[4];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("%-40s blocks %3d: %.2f cycles/DMMA\n", name, blocks, (double)h[0] / (reps * KS * 4 * (V == 9 ? 2 : 1)));
}
int main() {
  double2* gf; long long* d; double* s;
  cudaMalloc(&gf, 16 * 16 * 32 * 16); cudaMemset(gf, 0, 16 * 16 * 32 * 16);
  cudaMalloc(&d, 64); cudaMalloc(&s, 148 * 128 * 8);
  for (int b : {1, 148}) {
    run<0>("B from LDS.128, A in registers", gf, d, s, b);
    run<1>("B from LDS.128, rolling LDG of A", gf, d, s, b);
    run<2>("B from registers", gf, d, s, b);
    run<3>("B from LDS.128, prefetch distance 1", gf, d, s, b);
    run<4>("B from LDS.128, prefetch distance 2", gf, d, s, b);
    run<5>("B from LDS.128, prefetch distance 3", gf, d, s, b);
    run<9>("joint head: B shared by two A sets", gf, d, s, b);
  }
  return 0;
}

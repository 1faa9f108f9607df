// TMEM as the home of the HALS sweep's H tile (round 2 design probe).
//  (1) layout: what tcgen05.ld.16x256b returns to each thread after 32x32b stores with
//      value = lane*1000 + column (checks the "lane = column, 4 rows per 256-bit chunk" plan:
//      thread (gi = t/4, gt = t%4) should see lane gi's double #gt and lane gi+8's double #gt).
//  (2) DMMA.8x8x4 issue rate, one warp per SM sub-partition, 4 tiles × 2 k-steps per step
//      (16 DMMA), B fragments from: registers / LDS.128 / tcgen05.ld 16x256b (plain and
//      software-pipelined).
//  (3) row-warp TMEM round trip: 32x32b.x16 ld + wait, st + wait (latency).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void ld256x2(uint32_t ta, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(ta));
}
__device__ __forceinline__ void ld256x1(uint32_t ta, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(ta));
}
__device__ __forceinline__ void ld32x16(uint32_t ta, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(ta));
}
__device__ __forceinline__ void st32x16(uint32_t ta, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(ta),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// MODE 0: B in registers; 1: LDS.128; 2: tcgen05.ld then wait; 3: tcgen05.ld pipelined one step ahead
template <int MODE>
__global__ void __launch_bounds__(128, 1) rate(int steps, long long* out, double* sink, int* layout) {
  __shared__ __align__(16) double Hs[4][40 * 32];
  __shared__ uint32_t tb_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4 * 40 * 32; i += 128) (&Hs[0][0])[i] = 1.0 + 1e-3 * (i & 63);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tb_s))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tb = tb_s;
  const uint32_t tq = tb + ((uint32_t)(32 * warp) << 16);   // this warp's lane quarter
  // fill: lane L of the quarter, column c: value L*1000 + c
  for (int c0 = 0; c0 < 512; c0 += 16) {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = lane * 1000 + c0 + i;
    st32x16(tq + c0, v);
  }
  st_wait();
  if (blockIdx.x == 0 && warp == 1 && MODE == 2) {
    uint32_t v[8];
    ld256x2(tq + 8, v);
    ld_wait();
    for (int i = 0; i < 8; ++i) layout[lane * 8 + i] = (int)v[i];
    uint32_t w[4];
    ld256x1(tq + (16u << 16), w);
    ld_wait();
    for (int i = 0; i < 4; ++i) layout[256 + lane * 4 + i] = (int)w[i];
  }
  __syncwarp();
  double A[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) A[i] = 0.5 + 1e-3 * (lane + i);
  double acc[4][2] = {};
  double bv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) bv[i] = 1.0 + 1e-3 * i;
  const double* hs = Hs[warp];
  uint32_t nx[2][8];
  if (MODE == 3) {
    ld256x2(tq, nx[0]);
    ld256x2(tq + (16u << 16), nx[1]);
    ld_wait();
  }
  __syncwarp();
  const long long t0 = clock64();
#pragma unroll 1
  for (int s = 0; s < steps; ++s) {
    const int j = s & 15;
    if (MODE == 1) {
      const double2* p = reinterpret_cast<const double2*>(hs + ((8 * j) & 31) * 32 + (lane & 3) * 32 + 4 * (lane >> 2));
      const double2 a = p[0], b = p[1], c = p[64], d = p[65];
      bv[0] = a.x; bv[1] = a.y; bv[2] = b.x; bv[3] = b.y; bv[4] = c.x; bv[5] = c.y; bv[6] = d.x; bv[7] = d.y;
    } else if (MODE == 2) {
      uint32_t u[8], w[8];
      ld256x2(tq + 16 * j, u);
      ld256x2(tq + (16u << 16) + 16 * j, w);
      ld_wait();
      bv[0] = __hiloint2double(u[1], u[0]); bv[1] = __hiloint2double(u[3], u[2]);
      bv[2] = __hiloint2double(w[1], w[0]); bv[3] = __hiloint2double(w[3], w[2]);
      bv[4] = __hiloint2double(u[5], u[4]); bv[5] = __hiloint2double(u[7], u[6]);
      bv[6] = __hiloint2double(w[5], w[4]); bv[7] = __hiloint2double(w[7], w[6]);
    } else if (MODE == 3) {
      bv[0] = __hiloint2double(nx[0][1], nx[0][0]); bv[1] = __hiloint2double(nx[0][3], nx[0][2]);
      bv[2] = __hiloint2double(nx[1][1], nx[1][0]); bv[3] = __hiloint2double(nx[1][3], nx[1][2]);
      bv[4] = __hiloint2double(nx[0][5], nx[0][4]); bv[5] = __hiloint2double(nx[0][7], nx[0][6]);
      bv[6] = __hiloint2double(nx[1][5], nx[1][4]); bv[7] = __hiloint2double(nx[1][7], nx[1][6]);
      const int jn = (s + 1) & 15;
      ld256x2(tq + 16 * jn, nx[0]);
      ld256x2(tq + (16u << 16) + 16 * jn, nx[1]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) dmma(acc[t][0], acc[t][1], A[t], bv[t]);
#pragma unroll
    for (int t = 0; t < 4; ++t) dmma(acc[t][0], acc[t][1], A[4 + t], bv[4 + t]);
#pragma unroll
    for (int t = 0; t < 4; ++t) dmma(acc[t][0], acc[t][1], A[t], bv[4 + t]);
#pragma unroll
    for (int t = 0; t < 4; ++t) dmma(acc[t][0], acc[t][1], A[4 + t], bv[t]);
    if (MODE == 3) ld_wait();
  }
  const long long t1 = clock64();
  double sum = 0;
  for (int t = 0; t < 4; ++t) sum += acc[t][0] + acc[t][1];
  sink[blockIdx.x * 128 + threadIdx.x] = sum;
  if (blockIdx.x == 0 && lane == 0) out[warp] = t1 - t0;
  // (3) row-warp round trip: ld 16 columns, wait, st them back + 1, wait
  if (MODE == 2) {
    __syncwarp();
    const long long r0 = clock64();
    uint32_t v[16];
#pragma unroll 1
    for (int it = 0; it < 64; ++it) {
      ld32x16(tq + 16 * (it & 15), v);
      ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += 1;
      st32x16(tq + 16 * (it & 15), v);
      st_wait();
    }
    const long long r1 = clock64();
    if (blockIdx.x == 0 && lane == 0) out[4 + warp] = r1 - r0;
    sink[blockIdx.x * 128 + threadIdx.x] += v[lane & 15];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
  }
}

int main() {
  long long* out;
  double* sink;
  int* layout;
  cudaMallocManaged(&out, 8 * sizeof(long long));
  cudaMalloc(&sink, 148 * 128 * sizeof(double));
  cudaMallocManaged(&layout, 512 * sizeof(int));
  const int steps = 4096;
  const char* names[4] = {"B in registers", "B via LDS.128 (4 per 16 DMMA)", "B via tcgen05.ld 16x256b.x2 x2 + wait",
                          "B via tcgen05.ld, pipelined one step ahead"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (mode) {
        case 0: rate<0><<<148, 128>>>(steps, out, sink, layout); break;
        case 1: rate<1><<<148, 128>>>(steps, out, sink, layout); break;
        case 2: rate<2><<<148, 128>>>(steps, out, sink, layout); break;
        case 3: rate<3><<<148, 128>>>(steps, out, sink, layout); break;
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    }
    printf("%-45s %6.2f cycles per DMMA (warp 0), %6.2f (warp 3)\n", names[mode], out[0] / (16.0 * steps),
           out[3] / (16.0 * steps));
    if (mode == 2) printf("row-warp TMEM round trip (32x32b.x16 ld+wait+st+wait): %.1f cycles\n", out[4] / 64.0);
  }
  printf("layout 16x256b.x2 at (quarter 1, lane +0, col 8): thread: 8 words (lane*1000+col)\n");
  for (int t = 0; t < 32; ++t) {
    printf("  t%2d:", t);
    for (int i = 0; i < 8; ++i) printf(" %6d", layout[t * 8 + i]);
    printf("\n");
  }
  printf("layout 16x256b.x1 at (quarter 1, lane +16, col 0):\n");
  for (int t = 0; t < 32; ++t) {
    printf("  t%2d:", t);
    for (int i = 0; i < 4; ++i) printf(" %6d", layout[256 + t * 4 + i]);
    printf("\n");
  }
  return 0;
}

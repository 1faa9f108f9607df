// tcgen05.mma kind::i8 with A in tensor memory (TS form), M=128, N=16, K=32 per
// instruction: the shape a blocked Gauss-Seidel HALS sweep would use on the INT8 tensor
// cores (A = 128 columns of H × 128 rows, B = 16 Gram rows).  Checks the product against
// the host and measures cycles per MMA (one CTA).  Round-2 design probe.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo & 0x3FFFF) >> 4) << 16;
  d |= (uint64_t)((sbo & 0x3FFFF) >> 4) << 32;
  d |= (uint64_t)1 << 46;          // version 1 (sm_100)
  return d;                        // base offset 0, SWIZZLE_NONE (layout type 0)
}

constexpr int M = 128, N = 16, K = 128;

__global__ void __launch_bounds__(128, 1) probe(const int8_t* A, const int8_t* B, int* D, long long* cyc, int reps, int nacc) {
  __shared__ __align__(1024) int8_t Bs[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B (N × K, K-major) in core matrices of 8 rows × 16 bytes: core (g, c) at (g·(K/16) + c)·128
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K;
    const int g = n / 8, r = n % 8, c = k / 16, e = k % 16;
    Bs[(g * (K / 16) + c) * 128 + r * 16 + e] = B[n * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");   // Bs visible to the async (tensor) proxy
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tmem_base;
  const uint32_t a_tmem = tb;            // columns [0, 32): A, 4 int8 per 32-bit column
  const uint32_t d_tmem = tb + 32;       // columns [32, 48): D (int32)
  // A row m = lane m of TMEM: warp w writes lanes 32w..32w+31
  {
    const int m = warp * 32 + lane;
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = *reinterpret_cast<const uint32_t*>(A + m * K + 4 * j);
    const uint32_t addr = a_tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // instruction descriptor: D s32, A/B signed int8, K-major both, N>>3, M>>4
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    uint64_t bd[K / 32];
    for (int kc = 0; kc < K / 32; ++kc) bd[kc] = make_desc(smem_u32(Bs) + kc * 2 * 128, 128, (K / 16) * 128);
    t0 = clock64();
#pragma unroll 1
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int kc = 0; kc < K / 32; ++kc) {
        const uint32_t acc = (rep > 0 || kc > 0) ? 1u : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= nacc) break;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem + j * 16),
              "r"(a_tmem + kc * 8), "l"(bd[kc]), "r"(idesc), "r"(acc));
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)));
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)));
    }
  }
  if (tid == 0) { t1 = clock64(); cyc[0] = t1 - t0; }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // D: lanes = rows m, 16 columns
  {
    uint32_t v[16];
    const uint32_t addr = d_tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    const int m = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) D[m * N + j] = (int)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tb));
}

int main() {
  int8_t *hA = (int8_t*)malloc(M * K), *hB = (int8_t*)malloc(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (int8_t)(rand() % 255 - 127);
  for (int i = 0; i < N * K; ++i) hB[i] = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB; int* dD; long long* dc;
  cudaMalloc(&dA, M * K); cudaMalloc(&dB, N * K); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, hA, M * K, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, N * K, cudaMemcpyHostToDevice);
  for (int nacc : {1, 4, 8})
  for (int reps : {64, 1024}) {
    probe<<<1, 128>>>(dA, dB, dD, dc, reps, nacc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    int* hD = (int*)malloc(M * N * 4); long long hc;
    cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost); cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        long long ref = 0;
        for (int k = 0; k < K; ++k) ref += (long long)hA[m * K + k] * hB[n * K + k];
        ref *= (long long)((reps * (K / 32) + nacc - 1) / nacc) * 0 + 1;   // (checked only for nacc = 1)
        if (nacc == 1 && (int)(ref * reps) != hD[m * N + n]) ++bad;
      }
    printf("nacc %d reps %5d: %ld mismatches of %d, %lld cycles = %.2f cycles per MMA (M=128 N=16 K=32, A in TMEM)\n",
           nacc, reps, bad, M * N, hc, (double)hc / (reps * (K / 32) * nacc));
    free(hD);
  }
  return 0;
}

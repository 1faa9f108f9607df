// CTA-pair (cta_group::2) kind::i8 MMA as the INT8-digit product needs it (round 2 design probe):
//   D_cta (128 lanes × N=128, int32, each CTA's TMEM) = A_cta (128 × 32, the CTA's own smem tile,
//   different content per CTA at the SAME smem offset) · Bᵀ, B = 128 rows × 32 split 64 / 64 over
//   the two CTAs' smem.  Checks the result against the host and times back-to-back MMAs
//   (cycles per MMA) for cta_group::2 M=256 N=128 vs cta_group::1 M=128 N=128, both SS.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../paper_1805_06604_b200/csrc/tc.cuh"

__device__ __forceinline__ int off(int r, int kh) { return ((r >> 3) * 2 + kh) * 128 + (r & 7) * 16; }
__device__ __forceinline__ uint32_t mapa0(uint32_t a) {   // CTA 0's shared::cluster address of a
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(a));
  return r;
}

template <int MODE>   // 0: verify, 1: time cta_group::2, 2: time cta_group::1 (N = 128)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const int8_t* Ag, const int8_t* Bg, int* Dout, int iters, long long* cyc) {
  __shared__ __align__(1024) int8_t sA[4096];
  __shared__ __align__(1024) int8_t sB[4096];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb_s;
  const int rank = (int)tc::cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A: row i, byte k -> canonical layout; this CTA's A = rows [128·rank, 128·rank+128) of Ag (256 × 32)
  for (int e = threadIdx.x; e < 128 * 32; e += 128) {
    const int i = e / 32, k = e % 32;
    sA[off(i, k >> 4) + (k & 15)] = Ag[(128 * rank + i) * 32 + k];
  }
  // B: this CTA holds rows [64·rank, 64·rank + 64) (cta_group::2); all 128 rows for MODE 2
  for (int e = threadIdx.x; e < 128 * 32; e += 128) {
    const int j = e / 32, k = e % 32;
    if (MODE == 2 || j < 64) sB[off(j, k >> 4) + (k & 15)] = Bg[((MODE == 2 ? 0 : 64 * rank) + j) * 32 + k];
  }
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    if (MODE == 2) tc::tmem_alloc<128>(&tb_s);
    else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(tc::smem_u32(&tb_s))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
  }
  tc::fence_before();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tb = tb_s;
  const uint64_t dA = tc::desc_noswz(tc::smem_u32(sA), 128, 256);
  const uint64_t dB = tc::desc_noswz(tc::smem_u32(sB), 128, 256);
  long long t0 = 0, t1 = 0;
  if (MODE != 2 && rank == 0 && threadIdx.x == 0) {
    constexpr uint32_t ID = tc::idesc_i8(256, 128);
    t0 = clock64();
    for (int it = 0; it < iters; ++it)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tb),
          "l"(dA), "l"(dB), "r"(ID), "r"(it > 0 ? 1u : 0u)
          : "memory");
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                     tc::smem_u32(&bar)),
                 "h"((uint16_t)3)
                 : "memory");
  }
  if (MODE == 2 && threadIdx.x == 0) {
    constexpr uint32_t ID = tc::idesc_i8(128, 128);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) tc::mma_i8(tb, dA, dB, ID, it > 0 ? 1u : 0u);
    tc::commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after();
  if (threadIdx.x == 0) t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[MODE] = t1 - t0;
  // D: lane = A row (this CTA), column j = B row
  for (int j0 = 0; j0 < 128; j0 += 16) {
    uint32_t v[16];
    tc::ld16(tb + ((uint32_t)(32 * warp) << 16) + j0, v);
    tc::ld_wait();
    if (blockIdx.x < 2)
      for (int t = 0; t < 16; ++t) Dout[((long)(128 * rank + 32 * warp + lane)) * 128 + j0 + t] = (int)v[t];
  }
  tc::fence_before();
  tc::cluster_sync();
  if (warp == 0) {
    tc::fence_after();
    if (MODE == 2) tc::tmem_dealloc<128>(tb);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;\n" ::"r"(tb));
  }
}

int main() {
  int8_t *A, *B;
  int* D;
  long long* cyc;
  cudaMallocManaged(&A, 256 * 32);
  cudaMallocManaged(&B, 128 * 32);
  cudaMallocManaged(&D, 256 * 128 * sizeof(int));
  cudaMallocManaged(&cyc, 4 * sizeof(long long));
  srand(1);
  for (int i = 0; i < 256 * 32; ++i) A[i] = (int8_t)(rand() % 256 - 128);
  for (int i = 0; i < 128 * 32; ++i) B[i] = (int8_t)(rand() % 256 - 128);
  probe<0><<<2, 128>>>(A, B, D, 1, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("verify: %s\n", cudaGetErrorString(e)); return 1; }
  long bad = 0;
  for (int i = 0; i < 256; ++i)
    for (int j = 0; j < 128; ++j) {
      int s = 0;
      for (int k = 0; k < 32; ++k) s += A[i * 32 + k] * B[j * 32 + k];
      if (s != D[i * 128 + j]) ++bad;
    }
  printf("cta_group::2 M=256 N=128 K=32 kind::i8 (A per CTA, B split 64/64): %ld of %d wrong\n", bad, 256 * 128);
  const int iters = 4096;
  probe<1><<<148, 128>>>(A, B, D, iters, cyc);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("time2: %s\n", cudaGetErrorString(e)); return 1; }
  probe<2><<<148, 128>>>(A, B, D, iters, cyc);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("time1: %s\n", cudaGetErrorString(e)); return 1; }
  printf("cta_group::2 M=256 N=128: %.1f cycles per MMA (floor 64: 128x128x32 per SM)\n", (double)cyc[1] / iters);
  printf("cta_group::1 M=128 N=128: %.1f cycles per MMA (floor 64)\n", (double)cyc[2] / iters);
  return 0;
}

// tcgen05 kind::i8 issue-rate probe for the Ozaki digit GEMM shape (round 2 design probe).
// One "stage" = the 21 digit-pair MMAs of S = 6 levels (M = 128, N = BN, K = 32) into 6 level
// accumulators, operands resident in shared memory (no TMA), 148 CTAs.  Modes:
//   ss    : A and B from shared memory (SS form)
//   ts    : A from tensor memory (static, copied once), B from shared memory
//   tscp  : ts + the 6 A tiles copied shared → TMEM by tcgen05.cp every stage (double-buffered)
// Prints cycles per stage (ideal = 21 · 128·BN/256).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_1805_06604_b200/csrc/tc.cuh"

template <int BN, int MODE>
__global__ void __launch_bounds__(128, 1) probe(int stages, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;                  // 6 × 128 × 32
  uint8_t* sB = sm + 6 * 4096;       // 6 × BN × 32
  __shared__ uint32_t tb_s;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 6 * 4096 + 6 * BN * 32; i += 128) sm[i] = (uint8_t)(i * 37 + 11);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tb_s);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tb = tb_s;
  constexpr uint32_t ID = tc::idesc_i8(128, BN);
  if (threadIdx.x == 0) {
    const uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB);
    const uint32_t at0 = tb + 6 * BN;
    if (MODE != 0)
      for (int p = 0; p < 6; ++p) tc::cp_128x256b(at0 + p * 8, tc::desc_sw32(a0 + p * 4096));
    const long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
      const uint32_t at = at0 + (MODE == 2 ? (s & 1) * 48 : 0);
      if (MODE == 2)
        for (int p = 0; p < 6; ++p) tc::cp_128x256b(at + p * 8, tc::desc_sw32(a0 + p * 4096));
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const uint64_t bd = tc::desc_sw32(b0 + q * BN * 32);
#pragma unroll
        for (int p = 0; p < 6 - q; ++p) {
          if (MODE == 0) tc::mma_i8(tb + (p + q) * BN, tc::desc_sw32(a0 + p * 4096), bd, ID, 1u);
          else tc::mma_i8_ts(tb + (p + q) * BN, at + p * 8, bd, ID, 1u);
        }
      }
    }
    tc::commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) { tc::fence_after(); tc::tmem_dealloc<512>(tb); }
}

// level-split stage (3-CTA design): 7 MMAs into 2 accumulators (levels {0,5}: (0,0) and the six
// (p, 5-p)), SS form, B tiles BN rows; one CTA
template <int BN>
__global__ void __launch_bounds__(128, 1) probe_split(int stages, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;
  uint8_t* sB = sm + 6 * 4096;
  __shared__ uint32_t tb_s;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 6 * 4096 + 6 * BN * 32; i += 128) sm[i] = (uint8_t)(i * 37 + 11);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tb_s);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tb = tb_s;
  constexpr uint32_t ID = tc::idesc_i8(128, BN);
  if (threadIdx.x == 0) {
    const uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB);
    const long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
      tc::mma_i8(tb, tc::desc_sw32(a0), tc::desc_sw32(b0), ID, 1u);
#pragma unroll
      for (int p = 0; p < 6; ++p)
        tc::mma_i8(tb + BN, tc::desc_sw32(a0 + p * 4096), tc::desc_sw32(b0 + (5 - p) * BN * 32), ID, 1u);
    }
    tc::commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) { tc::fence_after(); tc::tmem_dealloc<512>(tb); }
}

template <int BN>
void run_split(long long* d) {
  const int smem = 6 * 4096 + 6 * BN * 32 + 1024;
  cudaFuncSetAttribute(probe_split<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 2000;
  probe_split<BN><<<148, 128, smem>>>(stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("split BN=%d: %s\n", BN, cudaGetErrorString(e)); return; }
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double ideal = 7.0 * 128 * BN / 256;
  printf("split BN=%3d: %8.1f cycles/stage (ideal %6.1f, %.0f%% of the i8 floor)\n", BN, (double)h / stages, ideal,
         100.0 * ideal / ((double)h / stages));
}

template <int BN, int MODE>
void run(const char* name, long long* d) {
  const int smem = 6 * 4096 + 6 * BN * 32 + 1024;
  cudaFuncSetAttribute(probe<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 2000;
  probe<BN, MODE><<<148, 128, smem>>>(stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s BN=%d: %s\n", name, BN, cudaGetErrorString(e)); return; }
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double ideal = 21.0 * 128 * BN / 256;
  printf("%-5s BN=%3d: %8.1f cycles/stage (ideal %6.1f, %.0f%% of the i8 floor)\n", name, BN, (double)h / stages, ideal,
         100.0 * ideal / ((double)h / stages));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 0>("ss", d); run<64, 1>("ts", d); run<64, 2>("tscp", d);
  run<80, 0>("ss", d);
  run<32, 0>("ss", d); run<32, 1>("ts", d); run<32, 2>("tscp", d);
  run_split<64>(d); run_split<96>(d); run_split<128>(d); run_split<160>(d); run_split<192>(d); run_split<256>(d);
  return 0;
}

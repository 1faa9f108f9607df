// tf32k.cuh — the TF32 variant's cross products on a hand-written tcgen05 kernel
// (kind::tf32, FP32 accumulation in TMEM), BASELINE configs[4]'s "TF32/FP32 variant".
//
// out (R × N) = A (R × K) · Bᵀ with B = X's rows (T·Xᵀ) or X's columns (W_yᵀX), both
// operands rounded to nearest TF32 and stored as the shared-memory images of their MMA
// tiles — K-major, no swizzle: for K chunk c (32 elements = 128 B) and row tile t, the rows ×
// 128 B image ordered [8-row group][K core matrix (8 of 16 B)][8 rows][16 B] — so each stage
// of an operand is ONE contiguous bulk copy (TMA engine).  M = 128 factor rows, N = 256 X rows,
// K = 8 per tcgen05.mma.kind::tf32; the X stream is read once per product (the variant is
// HBM-bound: 4 B·m·n per product).  K is cut into splits so the persistent grid is balanced;
// each split's FP32 tile goes to a partial buffer and `tf32_finish` adds them in FP64 in order.
// Roles as in ozk.cuh: warp 0 producer, warp 1 MMA issuer, warps 2-5 epilogue; accumulators
// double-buffered (2 × 256 TMEM columns).
#pragma once

#include <cstdint>

#include "common.cuh"
#include "tc.cuh"

namespace tf32k {

constexpr int KE = 32;                       // K elements per chunk (128 B)
constexpr int AROWS = 128, BROWS = 256;      // M and N of a tile
constexpr int A_TILE = AROWS * KE * 4, B_TILE = BROWS * KE * 4;   // 16 KB, 32 KB
constexpr int STAGE = A_TILE + B_TILE;
constexpr int NS = 4;
constexpr int SMEM = 1024 + NS * STAGE + 1024;
constexpr int THREADS = 192;
constexpr int ACC_COLS = BROWS;              // fp32 accumulator: 128 lanes × 256 columns

// byte offset of element (row, k) of an operand in its tile-image layout (rows per tile RT)
ENMF_DEV long img_off(long ntiles, int RT, long row, long k) {
  const long c = k / KE, t = row / RT;
  const int r = (int)(row % RT), kk = (int)(k % KE);
  return (c * ntiles + t) * (long)RT * KE * 4 + (long)(((r >> 3) * 8 + (kk >> 2)) * 8 + (r & 7)) * 16 + (kk & 3) * 4;
}

ENMF_DEV float to_tf32(double v) {
  // round to the nearest TF32 value: the tensor cores drop the low 13 bits of an FP32 operand
  // (a bias of half a TF32 ulp that the trace-identity error would amplify)
  const float f = (float)v;
  unsigned t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(f));
  return __uint_as_float(t);
}

// rows × K (row-major, lda) → tile images with RT rows per tile; the K padding of the last chunk is
// written as zeros (the buffer is shared by products of different K), padding rows stay zero
__global__ void pack_rows(const double* __restrict__ a, long rows, long K, long lda, int RT, float* __restrict__ out,
                          const DevState* st) {
  if (st && !dev_active(st)) return;
  const long nt = (rows + RT - 1) / RT;
  const long Kp = (K + KE - 1) / KE * KE;
  const long total = rows * Kp;
  char* o = reinterpret_cast<char*>(out);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const long r = i / Kp, k = i - r * Kp;
    *reinterpret_cast<float*>(o + img_off(nt, RT, r, k)) = k < K ? to_tf32(a[r * lda + k]) : 0.0f;
  }
}
// the columns of x (R × C, row-major) as the rows of the operand (C rows, K = R): coalesced
// reads along a row of x, one 4-byte store per element
__global__ void pack_cols(const double* __restrict__ x, long R, long C, int RT, float* __restrict__ out) {
  const long nt = (C + RT - 1) / RT;
  const long total = R * C;
  char* o = reinterpret_cast<char*>(out);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const long k = i / C, j = i - k * C;
    *reinterpret_cast<float*>(o + img_off(nt, RT, j, k)) = to_tf32(x[i]);
  }
}

struct Args {
  const float* A;    // factor images (nta row tiles of 128)
  const float* B;    // X images (ntb row tiles of 256)
  int nta, ntb;
  int R, N, nkc;     // rows, columns, 32-chunks of K
  int split_chunks, nks;   // chunks per K split, K splits
  float* part;       // nks × R × N
  const DevState* st;
};

__global__ void __launch_bounds__(THREADS, 1) gemm(Args g) {
  if (g.st && !dev_active(g.st)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + NS * A_TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;
  uint64_t* tfull = bars + 2 * NS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(tfull + b, 1);
      tc::mbar_init(tempty + b, 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc<512>(tbase_s);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *tbase_s;
  const int mt = (g.R + AROWS - 1) / AROWS;
  const int items = g.nks * mt * g.ntb;

  if (warp == 0) {                                     // ---- producer
    int stage = 0;
    uint32_t phase = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      const int ks = w / (mt * g.ntb), rem = w % (mt * g.ntb), mb = rem / g.ntb, tn = rem % g.ntb;
      const int c0 = ks * g.split_chunks, c1 = min(g.nkc, c0 + g.split_chunks);
      for (int c = c0; c < c1; ++c) {
        tc::mbar_wait(empty + stage, phase ^ 1);
        if (tc::elect_one()) {
          tc::mbar_expect_tx(full + stage, STAGE);
          tc::bulk_load(sA + stage * A_TILE, reinterpret_cast<const char*>(g.A) + ((long)c * g.nta + mb) * A_TILE,
                        A_TILE, full + stage);
          tc::bulk_load(sB + stage * B_TILE, reinterpret_cast<const char*>(g.B) + ((long)c * g.ntb + tn) * B_TILE,
                        B_TILE, full + stage);
        }
        __syncwarp();
        if (++stage == NS) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {                              // ---- MMA issuer
    constexpr uint32_t IDESC = tc::idesc_tf32(AROWS, BROWS);
    // K-adjacent core matrices 128 B apart, 8-row groups 8 × 128 B apart; one MMA = K 8 = 2 cores
    const uint64_t dA0 = tc::desc_noswz(tc::smem_u32(sA), 128, 1024);
    const uint64_t dB0 = tc::desc_noswz(tc::smem_u32(sB), 128, 1024);
    int stage = 0, ab = 0;
    uint32_t phase = 0, aph[2] = {0, 0};
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      const int ks = w / (mt * g.ntb);
      const int c0 = ks * g.split_chunks, c1 = min(g.nkc, c0 + g.split_chunks);
      tc::mbar_wait(tempty + ab, aph[ab] ^ 1);
      tc::fence_after();
      const uint32_t d = tbase + (uint32_t)(ab * ACC_COLS);
      for (int c = c0; c < c1; ++c) {
        tc::mbar_wait(full + stage, phase);
        tc::fence_after();
        const uint64_t dA = dA0 + (uint64_t)((stage * A_TILE) >> 4);
        const uint64_t dB = dB0 + (uint64_t)((stage * B_TILE) >> 4);
        const uint32_t first = c > c0 ? 1u : 0u;
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < KE / 8; ++k)
            tc::mma_tf32(d, dA + (uint64_t)(k * (256 >> 4)), dB + (uint64_t)(k * (256 >> 4)), IDESC,
                         first | (k > 0 ? 1u : 0u));
          tc::commit(empty + stage);
        }
        __syncwarp();
        if (++stage == NS) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::commit(tfull + ab);
      __syncwarp();
      aph[ab] ^= 1;
      ab ^= 1;
    }
  } else {                                             // ---- epilogue: FP32 tile → partial buffer
    const int quarter = warp & 3;
    int ab = 0;
    uint32_t aph[2] = {0, 0};
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      const int ks = w / (mt * g.ntb), rem = w % (mt * g.ntb), mb = rem / g.ntb, tn = rem % g.ntb;
      tc::mbar_wait(tfull + ab, aph[ab]);
      tc::fence_after();
      const long row = (long)mb * AROWS + quarter * 32 + lane;
      const uint32_t taddr = tbase + (uint32_t)(ab * ACC_COLS) + ((uint32_t)(quarter * 32) << 16);
      float* prow = g.part + ((long)ks * g.R + row) * g.N;
#pragma unroll 1
      for (int j0 = 0; j0 < BROWS; j0 += 16) {
        uint32_t v[16];
        tc::ld16(taddr + (uint32_t)j0, v);
        tc::ld_wait();
        const long col0 = (long)tn * BROWS + j0;
        if (row < g.R && col0 < g.N) {
          if (col0 + 16 <= g.N && (g.N & 3) == 0) {
#pragma unroll
            for (int t = 0; t < 16; t += 4)
              __stcg(reinterpret_cast<float4*>(prow + col0 + t),
                     make_float4(__uint_as_float(v[t]), __uint_as_float(v[t + 1]), __uint_as_float(v[t + 2]),
                                 __uint_as_float(v[t + 3])));
          } else {
#pragma unroll
            for (int t = 0; t < 16; ++t)
              if (col0 + t < g.N) prow[col0 + t] = __uint_as_float(v[t]);
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(tempty + ab);
      aph[ab] ^= 1;
      ab ^= 1;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc<512>(tbase);
  }
}

// out (R × N, ldo) = Σ_ks part[ks] (FP64, in split order)
__global__ void finish(const float* __restrict__ part, int nks, long R, long N, double* __restrict__ out, long ldo,
                       const DevState* st) {
  if (st && !dev_active(st)) return;
  const long total = R * N;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < nks; ++k) acc += (double)__ldcs(part + (long)k * total + i);
    const long r = i / N, c = i - r * N;
    out[r * ldo + c] = acc;
  }
}

}  // namespace tf32k

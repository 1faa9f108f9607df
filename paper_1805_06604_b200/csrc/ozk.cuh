// ozk.cuh — the INT8-digit cross products on hand-written tcgen05 kernels.
//
// W_yᵀX and T·Xᵀ (linalg.hpp:67-83, 107-124) in FP64 accuracy from 8-bit digits
// (the splitting scheme of ozaki.cuh: every operand row scaled by a power of two into
// (-1/2, 1/2), D_0 ∈ [-128, 127] and offset digits d_p = D_p − 128, p ≥ 1), with all
// S(S+1)/2 digit pairs of an X tile formed in ONE kernel:
//
//   * both operands K-major in a chunked digit layout [K/32][SMAX][rows][32 bytes]:
//     one 4-D TMA box (32 B × rows × S digits × 1 chunk) lands a stage's S digit
//     tiles of an operand in shared memory as S SWIZZLE_32B K-major tiles, and reads
//     contiguous runs of rows·32 bytes per digit from HBM;
//   * M = 128 factor rows (r ≤ 128 per M block), N = BN = 64 X rows per tile, K = 32
//     per tcgen05.mma.kind::i8; the pairs (p, q) are summed per LEVEL ℓ = p + q in
//     TMEM (S accumulators of 128 lanes × BN int32 columns: 384 of 512 columns at S = 6),
//     so the digit products never leave the SM;
//   * K is cut into units of ≤ 8192 (256 chunks): a level sum over one unit is exact
//     in int32 (|d_p·d_q| ≤ 2^14, ≤ 7 pairs per level: < 2^30); the epilogue reads the
//     S level sums (tcgen05.ld), forms Σ_ℓ 2^{-8ℓ} L_ℓ in FP64 and writes one FP64
//     partial per unit;
//   * `finish` adds the unit partials in fixed order, the exact offset corrections
//     (c_q·rowsum(d^A_p) + c_p·colsum(d^B_q) + c_p·c_q·K, from the digit sums along the
//     contracted index) and the truncation-bias estimate of ozaki::combine, and scales
//     by the two exponents.
//
// Warp roles (persistent, one CTA per SM, units kq-major so the CTAs in flight read
// the same factor chunk from L2): warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA
// issuer, warps 2-5 = epilogue (TMEM lane quarter = warp % 4).
#pragma once

#include <cstdint>

#include "common.cuh"
#include "ozaki.cuh"
#include "tc.cuh"

namespace ozk {

constexpr int SMAX = ozaki::SMAX;   // digits cut per operand
constexpr int KC = 32;              // bytes (= int8 elements) of K per chunk / per MMA
constexpr int UNIT_CHUNKS = 512;    // K per unit ≤ 16384: level sums exact in int32 (≤ 7 pairs · 2^14 · 2^14 < 2^31)
constexpr int EPI_THREADS = 128;
constexpr int THREADS = 64 + EPI_THREADS;
constexpr int SMEM_LIMIT = 232448;  // sm_100 opt-in dynamic shared memory per block
constexpr int PF = 12;              // stages of L2 prefetch ahead of the shared-memory pipeline

// Digit operand layout = the shared-memory image of the MMA operand tiles: for K chunk c (32 of
// K) and row tile t (128 rows), the SMAX digit tiles are contiguous (SMAX × 4 KB), each the
// canonical no-swizzle K-major layout of 128 rows × 32 B: core matrices of 8 rows × 16 B
// ordered [row group (16)][K half (2)] — so one stage of an operand is ONE contiguous bulk copy.
constexpr int TROWS = 128;                  // rows per tile (M of the factor, N of the X tile)
constexpr int TILE = TROWS * KC;            // 4 KB
ENMF_DEV long tile_base(long ntiles, long row, long c, int q) { return ((c * ntiles + row / TROWS) * SMAX + q) * (long)TILE; }
ENMF_DEV int tile_off(int r, int kh) { return ((r >> 3) * 2 + kh) * 128 + (r & 7) * 16; }   // row r % 128, K half

// ---- digit cuts into the chunked layout ------------------------------------------
// 32 consecutive values v[0..31] (one chunk of one operand row) scaled by 2^-(e+1): the
// SMAX digit rows of 32 bytes each into their tiles (two 16-byte core-matrix rows); adds the digits
// into acc (valid elements only; the padding past K is stored as zero digits, which add
// nothing to any digit product and are not counted in the sums).
ENMF_DEV void cut_chunk(const double (&v)[32], int nvalid, double scale, int8_t* out, long rows, long row, long c,
                        int (&acc)[SMAX]) {
  uint32_t w[SMAX][8];
#pragma unroll
  for (int q = 0; q < SMAX; ++q)
#pragma unroll
    for (int t = 0; t < 8; ++t) w[q][t] = 0;
#pragma unroll
  for (int u = 0; u < 32; ++u) {
    int8_t dd[SMAX];
    int dig[SMAX];
    ozaki::cut8(v[u] * scale, dd, 1, dig);
    const bool ok = u < nvalid;
#pragma unroll
    for (int q = 0; q < SMAX; ++q) {
      acc[q] += ok ? dig[q] : 0;
      w[q][u >> 2] |= (ok ? (uint32_t)(uint8_t)dd[q] : 0u) << (8 * (u & 3));
    }
  }
  const long nt = (rows + TROWS - 1) / TROWS;
  const int r = (int)(row % TROWS);
#pragma unroll
  for (int q = 0; q < SMAX; ++q) {
    int8_t* t = out + tile_base(nt, row, c, q);
    *reinterpret_cast<uint4*>(t + tile_off(r, 0)) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
    *reinterpret_cast<uint4*>(t + tile_off(r, 1)) = make_uint4(w[q][4], w[q][5], w[q][6], w[q][7]);
  }
}

ENMF_DEV double pow2_neg(int e1) { return __longlong_as_double((long long)(1023 - e1) << 52); }   // 2^-e1

// Row-scaled operand: `rows` rows of a (row-major, lda), exponent per row from e_row (or, when
// amax != nullptr, from the row's |max| bit pattern — the per-product factor path, which also
// publishes the exponent into e_row).  Thread = (row, chunk group); grid.x over row blocks of
// blockDim.x, grid.y over chunk groups.  sums[q·rows + row] (zeroed by the caller) += digit sums.
__global__ void split_rows_chunked(const double* __restrict__ a, long rows, long K, long lda, int* e_row,
                                   const unsigned long long* amax, int8_t* __restrict__ out, int* __restrict__ sums,
                                   const DevState* st) {
  if (st && !dev_active(st)) return;
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  int e;
  if (amax) {
    e = ozaki::exp_above(__longlong_as_double((long long)amax[row]));
    if (blockIdx.y == 0) e_row[row] = e;
  } else {
    e = e_row[row];
  }
  const double scale = pow2_neg(e + 1);
  const long nkc = (K + KC - 1) / KC;
  const double* ar = a + row * lda;
  const bool vec = ((reinterpret_cast<uintptr_t>(ar) & 15) == 0);
  int acc[SMAX] = {};
  for (long c = blockIdx.y; c < nkc; c += gridDim.y) {
    const long k0 = c * KC;
    const int nvalid = (int)min((long)KC, K - k0);
    double v[32];
    if (vec && nvalid == KC) {
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(ar + k0) + h);
        v[2 * h] = t.x;
        v[2 * h + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = u < nvalid ? ar[k0 + u] : 0.0;
    }
    cut_chunk(v, nvalid, scale, out, rows, row, c, acc);
  }
#pragma unroll
  for (int q = 0; q < SMAX; ++q) atomicAdd(sums + (long)q * rows + row, acc[q]);
}

// Column-scaled operand: the rows of the digit matrix are the COLUMNS j of x (R × C,
// row-major, ld), contracted over x's rows; exponent per column e_col[j].  Thread = (column,
// chunk group): each chunk reads 32 rows of one column (coalesced across the warp) and
// writes 32 contiguous bytes per digit.  sums[q·C + j] += digit sums.
__global__ void split_cols_chunked(const double* __restrict__ x, long R, long C, long ld, const int* __restrict__ e_col,
                                   int8_t* __restrict__ out, int* __restrict__ sums) {
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= C) return;
  const double scale = pow2_neg(e_col[j] + 1);
  const long nkc = (R + KC - 1) / KC;
  int acc[SMAX] = {};
  for (long c = blockIdx.y; c < nkc; c += gridDim.y) {
    const long i0 = c * KC;
    const int nvalid = (int)min((long)KC, R - i0);
    double v[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = u < nvalid ? __ldcs(x + (i0 + u) * ld + j) : 0.0;
    cut_chunk(v, nvalid, scale, out, C, j, c, acc);
  }
#pragma unroll
  for (int q = 0; q < SMAX; ++q) atomicAdd(sums + (long)q * C + j, acc[q]);
}

// ---- the digit GEMM ---------------------------------------------------------------
// The S(S+1)/2 digit pairs of a tile are split BY LEVEL over the CL CTAs of a cluster: CTA
// rank ρ owns the levels of group ρ (the pairs (p, q) with p + q in the group) and keeps one
// 128-lane × BN accumulator per owned level in its TMEM.  With BN = 128 every MMA (M = 128,
// N = 128, K = 32) runs at the tensor core's floor — measured: an M = 128 kind::i8 MMA costs
// ≥ ~48 cycles whatever its N, so N = 64 tiles (all S levels in one CTA) reach only 67%
// (profiles/r02_umma_rate.txt) — and the groups are balanced:
//   S = 6, CL = 2: {0,1,2,4} (11 pairs) | {3,5} (10);   S = 6, CL = 3: {0,5} | {1,4} | {2,3} (7 each)
//   S = 7, CL = 2: {0,2,3,4} (13) | {1,5,6} (15);       S = 7, CL = 3: {1,6} | {2,5} | {0,3,4}
// Every digit tile of a stage (S factor tiles of 128 rows, S X tiles of BN rows, 32 B of K
// each) is loaded ONCE per cluster by one CTA and multicast to all CL of them.
template <int S, int CL>
struct Levels {
  static constexpr int G = CL;
  __host__ __device__ static constexpr int count(int rank) {
    return S == 6 ? (CL == 2 ? (rank == 0 ? 4 : 2) : 2) : (CL == 2 ? (rank == 0 ? 4 : 3) : (rank == 2 ? 3 : 2));
  }
  __host__ __device__ static constexpr int level(int rank, int i) {
    // tables above, row = rank, padded with -1
    return S == 6 ? (CL == 2 ? (rank == 0 ? (i == 0 ? 0 : i == 1 ? 1 : i == 2 ? 2 : 4) : (i == 0 ? 3 : 5))
                             : (rank == 0 ? (i == 0 ? 0 : 5) : rank == 1 ? (i == 0 ? 1 : 4) : (i == 0 ? 2 : 3)))
                  : (CL == 2 ? (rank == 0 ? (i == 0 ? 0 : i == 1 ? 2 : i == 2 ? 3 : 4) : (i == 0 ? 1 : i == 1 ? 5 : 6))
                             : (rank == 0 ? (i == 0 ? 1 : 6) : rank == 1 ? (i == 0 ? 2 : 5) : (i == 0 ? 0 : i == 1 ? 3 : 4)));
  }
  static constexpr int MAXL = S == 6 ? (CL == 2 ? 4 : 2) : (CL == 2 ? 4 : 3);
};

struct GemmArgs {
  const int8_t* A;   // factor digits (tile layout, nta row tiles)
  const int8_t* B;   // X digits (tile layout, ntb row tiles)
  int nta, ntb;
  int R, N;          // factor rows, X rows of the digit operands
  int nkc;           // 32-chunks of K (padded)
  int unit_chunks;   // chunks per unit (≤ UNIT_CHUNKS)
  int nkq, nmb, ntn; // units along K, M blocks of 128, N tiles of BN
  double* ws;        // CL × nkq × R × N FP64 partials (one slice per level group)
  const DevState* st;
};

template <int S, int CL, int BN>
struct Cfg {
  static_assert(BN == TROWS, "X tiles of 128 rows (the digit layout's row tile)");
  static constexpr int A_TILE = TILE, B_TILE = TILE;
  static constexpr int A_BYTES = S * A_TILE;
  static constexpr int B_BYTES = S * B_TILE;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int NS = (SMEM_LIMIT - 2048) / STAGE > 8 ? 8 : (SMEM_LIMIT - 2048) / STAGE;
  static constexpr int SMEM = 1024 + NS * STAGE + 1024;
  static constexpr int ACC_COLS = Levels<S, CL>::MAXL * BN;        // one accumulator set
  static constexpr int NACC = 2 * ACC_COLS <= 512 ? 2 : 1;        // double-buffered when it fits
  static constexpr int TMEM_COLS = NACC * ACC_COLS <= 256 ? 256 : 512;
  static_assert(ACC_COLS <= 512, "level accumulators must fit the 512 TMEM columns");
  static_assert(NS >= 3, "pipeline too shallow");
};

template <int S, int CL, int BN>
__global__ void __launch_bounds__(THREADS, 1) gemm_levels(GemmArgs g) {
  using C = Cfg<S, CL, BN>;
  using LV = Levels<S, CL>;
  if (g.st && !dev_active(g.st)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                  // NS × A_BYTES
  uint8_t* sB = smem + C::NS * C::A_BYTES;             // NS × B_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::NS * C::STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::NS;
  uint64_t* tfull = bars + 2 * C::NS;                  // [NACC]
  uint64_t* tempty = tfull + 2;                        // [NACC]
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)tc::cluster_rank();
  const int cluster = blockIdx.x / CL, nclusters = gridDim.x / CL;
  constexpr uint16_t MASK = (uint16_t)((1u << CL) - 1);
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NS; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, CL);                    // every CTA's MMA issuer frees the stage
    }
    for (int b = 0; b < C::NACC; ++b) {
      tc::mbar_init(tfull + b, 1);
      tc::mbar_init(tempty + b, EPI_THREADS);
    }
    tc::fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc<C::TMEM_COLS>(tbase_s);
  tc::fence_before();
  tc::cluster_sync();                                  // peers' barriers initialised before any multicast
  tc::fence_after();
  const uint32_t tbase = *tbase_s;

  const int items = g.nkq * g.nmb * g.ntn;
  if (warp == 0) {                                     // ---- TMA producer (this CTA's share of the tiles)
    int stage = 0;
    uint32_t phase = 0;
    // the stage = 2S contiguous 4 KB tiles (S factor, S X), this CTA's contiguous share of them
    // multicast to the cluster (A: tiles [0, S), B: [S, 2S))
    const int t0 = rank * 2 * S / CL, t1 = (rank + 1) * 2 * S / CL;
    const int ae = min(t1, S), b0t = max(t0, S) - S, b1t = t1 - S;
    for (int w = cluster; w < items; w += nclusters) {
      const int kq = w / (g.nmb * g.ntn), rem = w % (g.nmb * g.ntn);
      const int mb = rem / g.ntn, tn = rem % g.ntn;
      const int c0 = kq * g.unit_chunks, c1 = min(g.nkc, c0 + g.unit_chunks);
      for (int c = c0; c < c1; ++c) {
        tc::mbar_wait(empty + stage, phase ^ 1);       // every CTA of the cluster is done with the stage
        if (tc::elect_one()) {
          tc::mbar_expect_tx(full + stage, C::STAGE);
          const int8_t* asrc = g.A + ((long)c * g.nta + mb) * SMAX * TILE;
          const int8_t* bsrc = g.B + ((long)c * g.ntb + tn) * SMAX * TILE;
          if (t0 < S)
            tc::bulk_load_mc(sA + stage * C::A_BYTES + t0 * TILE, asrc + (long)t0 * TILE, (uint32_t)((ae - t0) * TILE),
                             full + stage, MASK);
          if (t1 > S) {
            tc::bulk_load_mc(sB + stage * C::B_BYTES + b0t * TILE, bsrc + (long)b0t * TILE,
                             (uint32_t)((b1t - b0t) * TILE), full + stage, MASK);
            // the X digits stream from HBM exactly once: pull the tiles PF stages ahead into L2 so
            // the (few-stage) shared-memory pipeline only sees L2 latency
            if (c + PF < c1)
              tc::bulk_prefetch_l2(g.B + ((long)(c + PF) * g.ntb + tn) * SMAX * TILE + (long)b0t * TILE,
                                   (uint32_t)((b1t - b0t) * TILE));
          }
        }
        __syncwarp();
        if (++stage == C::NS) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {                              // ---- MMA issuer (this CTA's levels)
    constexpr uint32_t IDESC = tc::idesc_i8(128, BN);
    // no-swizzle K-major descriptors: K-adjacent core matrices 128 B apart, 8-row groups 256 B
    const uint64_t dA0 = tc::desc_noswz(tc::smem_u32(sA), 128, 256);
    const uint64_t dB0 = tc::desc_noswz(tc::smem_u32(sB), 128, 256);
    int stage = 0, ab = 0;
    uint32_t phase = 0, aph[2] = {0, 0};
    const int nl = LV::count(rank);
    for (int w = cluster; w < items; w += nclusters) {
      const int kq = w / (g.nmb * g.ntn);
      const int c0 = kq * g.unit_chunks, c1 = min(g.nkc, c0 + g.unit_chunks);
      tc::mbar_wait(tempty + ab, aph[ab] ^ 1);         // the epilogue has drained this accumulator set
      tc::fence_after();
      const uint32_t dset = tbase + (uint32_t)(ab * C::ACC_COLS);
      for (int c = c0; c < c1; ++c) {
        tc::mbar_wait(full + stage, phase);
        tc::fence_after();
        const uint64_t dA = dA0 + (uint64_t)((stage * C::A_BYTES) >> 4);
        const uint64_t dB = dB0 + (uint64_t)((stage * C::B_BYTES) >> 4);
        const uint32_t first = c > c0 ? 1u : 0u;
        if (tc::elect_one()) {
#pragma unroll
          for (int i = 0; i < LV::MAXL; ++i) {
            if (i < nl) {
              const int l = LV::level(rank, i);
              const uint32_t d = dset + (uint32_t)(i * BN);
#pragma unroll
              for (int q = 0; q < S; ++q) {
                const int p = l - q;
                if (p >= 0 && p < S)
                  tc::mma_i8(d, dA + (uint64_t)(p * (TILE >> 4)), dB + (uint64_t)(q * (TILE >> 4)), IDESC,
                             (first | (q > 0 ? 1u : 0u)));
              }
            }
          }
          tc::commit_mc(empty + stage, MASK);          // frees the stage in every CTA of the cluster
        }
        __syncwarp();
        if (++stage == C::NS) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::commit(tfull + ab);     // this group's level sums of the unit complete
      __syncwarp();
      aph[ab] ^= 1;
      if (C::NACC == 2) ab ^= 1;
    }
  } else {                                             // ---- epilogue (warps 2..5)
    const int quarter = warp & 3;
    const int nl = LV::count(rank);
    int ab = 0;
    uint32_t aph[2] = {0, 0};
    for (int w = cluster; w < items; w += nclusters) {
      const int kq = w / (g.nmb * g.ntn), rem = w % (g.nmb * g.ntn);
      const int mb = rem / g.ntn, tn = rem % g.ntn;
      tc::mbar_wait(tfull + ab, aph[ab]);
      tc::fence_after();
      const long row = (long)mb * 128 + quarter * 32 + lane;
      const uint32_t taddr = tbase + (uint32_t)(ab * C::ACC_COLS) + ((uint32_t)(quarter * 32) << 16);
      double* wrow = g.ws + (((long)rank * g.nkq + kq) * g.R + row) * g.N;
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 16) {
        uint32_t v[LV::MAXL][16];
#pragma unroll
        for (int i = 0; i < LV::MAXL; ++i)
          if (i < nl) tc::ld16(taddr + (uint32_t)(i * BN + j0), v[i]);
        tc::ld_wait();
        const long col0 = (long)tn * BN + j0;
        if (row < g.R && col0 < g.N) {
          double o[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            double acc = 0.0;                          // Σ 2^{-8ℓ} L_ℓ over this group's levels
#pragma unroll
            for (int i = LV::MAXL - 1; i >= 0; --i)
              if (i < nl)
                acc = __dadd_rn(acc, __dmul_rn((double)(int)v[i][t],
                                               __longlong_as_double((long long)(1023 - 8 * LV::level(rank, i)) << 52)));
            o[t] = acc;
          }
          if (col0 + 16 <= g.N && ((g.N & 1) == 0)) {
#pragma unroll
            for (int t = 0; t < 16; t += 2)
              __stcg(reinterpret_cast<double2*>(wrow + col0 + t), make_double2(o[t], o[t + 1]));
          } else {
#pragma unroll
            for (int t = 0; t < 16; ++t)
              if (col0 + t < g.N) wrow[col0 + t] = o[t];
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(tempty + ab);
      aph[ab] ^= 1;
      if (C::NACC == 2) ab ^= 1;
    }
  }
  tc::fence_before();
  tc::cluster_sync();                                  // no CTA leaves while a peer may still signal it
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc<C::TMEM_COLS>(tbase);
  }
}

ENMF_DEV double p2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }   // 2^e, |e| < 1023

// out (R × N, row stride ldo) from the unit partials: Σ_kq ws[kq] + offset corrections per
// level + truncation-bias estimate (ozaki::combine's), scaled by 2^{ea_i + eb_j + 2 − 16}.
template <int S>
__global__ void __launch_bounds__(256) finish(const double* __restrict__ ws, int nparts, long R, long N, long K,
                                              const int* __restrict__ ea, const int* __restrict__ eb,
                                              const int* __restrict__ asum, const int* __restrict__ bsum,
                                              double* __restrict__ out, long ldo, const DevState* st) {
  if (st && !dev_active(st)) return;
  const long i = blockIdx.y;
  const int ei = ea[i];
  int as[S];
#pragma unroll
  for (int p = 0; p < S; ++p) as[p] = asum[(long)p * R + i];
  for (long j = (long)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (long)gridDim.x * blockDim.x) {
    int bs[S];
#pragma unroll
    for (int q = 0; q < S; ++q) bs[q] = bsum[(long)q * N + j];
    const int base = ei + eb[j] + 2;
    // truncation-bias estimate (ozaki::combine): dropped pairs p + q >= S from the digit sums,
    // uncut residuals uniform
    double ra[S], cb[S];
#pragma unroll
    for (int p = 0; p < S; ++p) {
      ra[p] = (double)as[p] + (p ? 128.0 * (double)K : 0.0);
      cb[p] = (double)bs[p] + (p ? 128.0 * (double)K : 0.0);
    }
    double corr = 0.0, sa = 0.0, sb = 0.0;
#pragma unroll
    for (int p = 1; p < S; ++p)
#pragma unroll
      for (int q = S - p; q < S; ++q) corr += (ra[p] * cb[q]) * p2(-8 * (p + q + 2));
    corr /= (double)K;
#pragma unroll
    for (int p = S - 1; p >= 0; --p) {
      sa += ra[p] * p2(-8 * (p + 1));
      sb += cb[p] * p2(-8 * (p + 1));
    }
    corr += (sa + sb) * p2(-8 * S - 1);
    // in units of 2^{base-16}: bias, then the exact offset corrections per level (smallest
    // weight first), then the digit-product partials of the K units in order
    double acc = corr * 65536.0;
#pragma unroll
    for (int l = S - 1; l >= 0; --l) {
      long long cl = 0;
#pragma unroll
      for (int q = 0; q <= l; ++q) {
        const int p = l - q;
        if (q) cl += 128LL * as[p];
        if (p) cl += 128LL * bs[q];
        if (p && q) cl += 16384LL * K;
      }
      acc += (double)cl * p2(-8 * l);
    }
    for (int u = 0; u < nparts; ++u) acc += __ldcs(ws + ((long)u * R + i) * N + j);   // groups × K units, in order
    const int e = base - 16;   // exact power-of-two scaling (ldexp outside the normal range)
    out[i * ldo + j] = (e > -1000 && e < 1000) ? acc * p2(e) : ldexp(acc, e);
  }
}

}  // namespace ozk

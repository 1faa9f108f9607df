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
constexpr int UNIT_CHUNKS = 256;    // K per unit ≤ 8192: level sums exact in int32
constexpr int EPI_THREADS = 128;
constexpr int THREADS = 64 + EPI_THREADS;
constexpr int SMEM_LIMIT = 232448;  // sm_100 opt-in dynamic shared memory per block

// byte offset of (row, k) digit plane q in the chunked layout [Kp/32][SMAX][rows][32]
ENMF_DEV long chunk_off(long rows, long row, long c, int q) { return ((c * SMAX + q) * rows + row) * KC; }

// ---- digit cuts into the chunked layout ------------------------------------------
// 32 consecutive values v[0..31] (one chunk of one operand row) scaled by 2^-(e+1): the
// SMAX digit rows of 32 bytes each at out + chunk_off(rows, row, c, q); adds the digits
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
#pragma unroll
  for (int q = 0; q < SMAX; ++q) {
    uint4* o = reinterpret_cast<uint4*>(out + chunk_off(rows, row, c, q));
    o[0] = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
    o[1] = make_uint4(w[q][4], w[q][5], w[q][6], w[q][7]);
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
struct GemmArgs {
  int R, N;          // factor rows, X rows of the digit operands
  int nkc;           // 32-chunks of K (padded)
  int unit_chunks;   // chunks per unit (≤ UNIT_CHUNKS)
  int nkq, nmb, ntn; // units along K, M blocks of 128, N tiles of BN
  double* ws;        // nkq × R × N FP64 partials
  const DevState* st;
};

template <int S, int BN>
struct Cfg {
  static constexpr int A_BYTES = S * 128 * KC;
  static constexpr int B_BYTES = S * BN * KC;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int NS = (SMEM_LIMIT - 2048) / STAGE > 8 ? 8 : (SMEM_LIMIT - 2048) / STAGE;
  static constexpr int SMEM = 1024 + NS * STAGE + 1024;
  static constexpr int TMEM_COLS = S * BN <= 256 ? 256 : 512;
  static_assert(S * BN <= 512, "levels × BN must fit the 512 TMEM columns");
  static_assert(NS >= 3, "pipeline too shallow");
};

template <int S, int BN>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_levels(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, GemmArgs g) {
  using C = Cfg<S, BN>;
  if (g.st && !dev_active(g.st)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                  // NS × A_BYTES
  uint8_t* sB = smem + C::NS * C::A_BYTES;             // NS × B_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::NS * C::STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::NS;
  uint64_t* tfull = bars + 2 * C::NS;
  uint64_t* tempty = tfull + 1;
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&ta);
    tc::prefetch_tmap(&tb);
    for (int s = 0; s < C::NS; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    tc::mbar_init(tfull, 1);
    tc::mbar_init(tempty, EPI_THREADS);
    tc::fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc<C::TMEM_COLS>(tbase_s);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *tbase_s;

  const int units = g.nkq * g.nmb * g.ntn;
  if (warp == 0) {
    if (lane == 0) {                                   // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int kq = u / (g.nmb * g.ntn), rem = u % (g.nmb * g.ntn);
        const int mb = rem / g.ntn, tn = rem % g.ntn;
        const int c0 = kq * g.unit_chunks, c1 = min(g.nkc, c0 + g.unit_chunks);
        for (int c = c0; c < c1; ++c) {
          tc::mbar_wait(empty + stage, phase ^ 1);
          tc::mbar_expect_tx(full + stage, C::STAGE);
          tc::tma_load_4d(sA + stage * C::A_BYTES, &ta, full + stage, 0, mb * 128, 0, c);
          tc::tma_load_4d(sB + stage * C::B_BYTES, &tb, full + stage, 0, tn * BN, 0, c);
          if (++stage == C::NS) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {                                   // ---- MMA issuer
      constexpr uint32_t IDESC = tc::idesc_i8(128, BN);
      int stage = 0;
      uint32_t phase = 0, aphase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int kq = u / (g.nmb * g.ntn);
        const int c0 = kq * g.unit_chunks, c1 = min(g.nkc, c0 + g.unit_chunks);
        tc::mbar_wait(tempty, aphase ^ 1);             // the epilogue has drained TMEM
        tc::fence_after();
        for (int c = c0; c < c1; ++c) {
          tc::mbar_wait(full + stage, phase);
          tc::fence_after();
          const uint32_t a0 = tc::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = tc::smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int q = 0; q < S; ++q) {
            const uint64_t bd = tc::desc_sw32(b0 + q * BN * KC);
#pragma unroll
            for (int p = 0; p < S - q; ++p)
              tc::mma_i8(tbase + (uint32_t)((p + q) * BN), tc::desc_sw32(a0 + p * 128 * KC), bd, IDESC,
                         (c > c0 || q > 0) ? 1u : 0u);
          }
          tc::commit(empty + stage);                   // frees the stage when these MMAs are done
          if (++stage == C::NS) { stage = 0; phase ^= 1; }
        }
        tc::commit(tfull);                             // level sums of the unit complete
        aphase ^= 1;
      }
    }
  } else {                                             // ---- epilogue (warps 2..5)
    const int quarter = warp & 3;
    uint32_t aphase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int kq = u / (g.nmb * g.ntn), rem = u % (g.nmb * g.ntn);
      const int mb = rem / g.ntn, tn = rem % g.ntn;
      tc::mbar_wait(tfull, aphase);
      tc::fence_after();
      const long row = (long)mb * 128 + quarter * 32 + lane;
      const uint32_t taddr = tbase + ((uint32_t)(quarter * 32) << 16);
      double* wrow = g.ws + ((long)kq * g.R + row) * g.N;
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 16) {
        uint32_t v[S][16];
#pragma unroll
        for (int l = 0; l < S; ++l) tc::ld16(taddr + (uint32_t)(l * BN + j0), v[l]);
        tc::ld_wait();
        const long col0 = (long)tn * BN + j0;
        if (row < g.R) {
          double o[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            double acc = 0.0;                          // Σ_ℓ 2^{-8ℓ} L_ℓ, smallest weight first
#pragma unroll
            for (int l = S - 1; l >= 0; --l)
              acc = __dadd_rn(acc, __dmul_rn((double)(int)v[l][t], __longlong_as_double((long long)(1023 - 8 * l) << 52)));
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
      tc::mbar_arrive(tempty);
      aphase ^= 1;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::fence_after();
    tc::tmem_dealloc<C::TMEM_COLS>(tbase);
  }
}

// out (R × N, row stride ldo) from the unit partials: Σ_kq ws[kq] + offset corrections per
// level + truncation-bias estimate (ozaki::combine's), scaled by 2^{ea_i + eb_j + 2 − 16}.
template <int S>
__global__ void __launch_bounds__(256) finish(const double* __restrict__ ws, int nkq, long R, long N, long K,
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
      for (int q = S - p; q < S; ++q) corr += ldexp(ra[p] * cb[q], -8 * (p + q + 2));
    corr /= (double)K;
#pragma unroll
    for (int p = S - 1; p >= 0; --p) {
      sa += ldexp(ra[p], -8 * (p + 1));
      sb += ldexp(cb[p], -8 * (p + 1));
    }
    corr += ldexp(sa + sb, -8 * S - 1);
    // in units of 2^{base-16}: bias, then the exact offset corrections per level (smallest
    // weight first), then the digit-product partials of the K units in order
    double acc = ldexp(corr, 16);
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
      acc += ldexp((double)cl, -8 * l);
    }
    for (int kq = 0; kq < nkq; ++kq) acc += __ldcs(ws + ((long)kq * R + i) * N + j);
    out[i * ldo + j] = ldexp(acc, base - 16);
  }
}

}  // namespace ozk

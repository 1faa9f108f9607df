// ozaki.cuh — FP64-accurate cross products on the B200's INT8 tensor cores.
//
// W_yᵀX and T·Xᵀ (linalg.hpp:67-124) are the two large contractions of an outer
// iteration (2·r·m·n flop each).  B200 runs FP64 on DMMA.8x8x4 at 37 TF/s but
// INT8 on tcgen05 at ~3 POP/s (profiles/r01_int8_probe.txt), so the products are
// computed by error-free splitting (Ozaki's scheme) with full 8-bit digits: every
// operand row is scaled by a power of two into (-1/2, 1/2) and cut into S digits of
// 8 bits,
//     a = 2^{e+1} · sum_{p<S} D_p · 2^{-8(p+1)},   D_0 = floor(256 z) ∈ [-128, 127],
//     D_p = floor(256 r_p) ∈ [0, 255] stored as d_p = D_p − 128 (p ≥ 1)   (exact cuts)
// so every stored digit is a signed int8 and the offsets c_p = 128 (p ≥ 1) come back as
// rank-one corrections from the digits' sums along the contracted index:
//     D^A_p·D^B_q = d^A_p·d^B_q + c_q·rowsum(d^A_p) + c_p·colsum(d^B_q) + c_p·c_q·K
// each d^A_p·d^B_q an int8×int8→int32 tensor-core GEMM (exact while K·128² < 2³¹),
// the corrections exact integers.  With S = 6 levels (21 digit GEMMs) the neglected
// terms are ~2^{-47} of the row maxima — below FP64 accumulation over K = 32768 — and
// the sum over the digit pairs is formed in FP64 smallest term first.  (7-bit digits,
// d ∈ [-127, 127] by truncation, need S = 7 levels = 28 GEMMs for the same accuracy.)  X's digits are cut once per load (X is
// fixed); the factor's digits once per product.  The digit GEMMs are grouped by
// X digit q: one GEMM multiplies the stacked factor digits p = 0..S-1-q (an
// (S-q)·r-row operand) by X digit q, so X is streamed S times per product.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace ozaki {

constexpr int SMAX = 7;                   // digits cut per operand (8 bits each)
// digit levels kept, S ∈ {6, 7}: products d_p·d_q with p + q < S (S(S+1)/2 of them).  6 levels
// for X with a narrow per-row / per-column dynamic range, 7 otherwise (ozaki_prepare_x)

// The SMAX digits of z ∈ (-1/2, 1/2) (exact: scaling by 256, floor and the subtraction
// are exact in FP64); plane stride dstride; returns the digits for row / column sums.
ENMF_DEV void cut8(double z, int8_t* o, long dstride, int (&dig)[SMAX]) {
  double t = z * 256.0;
  double d = floor(t);
  dig[0] = (int)d;                       // [-128, 127]
  o[0] = (int8_t)dig[0];
  t -= d;                                // [0, 1)
#pragma unroll
  for (int p = 1; p < SMAX; ++p) {
    t *= 256.0;
    d = floor(t);
    t -= d;
    dig[p] = (int)d - 128;               // [-128, 127]
    o[p * dstride] = (int8_t)dig[p];
  }
}

// block-wide sums of the SMAX per-thread digit sums, added into sums[p * stride]
ENMF_DEV void add_digit_sums(const int (&acc)[SMAX], int* sums, long stride) {
  __shared__ int sh[SMAX][32];
  int v[SMAX];
#pragma unroll
  for (int p = 0; p < SMAX; ++p) v[p] = __reduce_add_sync(0xffffffffu, acc[p]);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int p = 0; p < SMAX; ++p) sh[p][threadIdx.x >> 5] = v[p];
  __syncthreads();
  if (threadIdx.x < SMAX) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[threadIdx.x][w];
    atomicAdd(sums + threadIdx.x * stride, t);   // integer: order-independent, exact
  }
}

// largest |x| → exponent e with |x| / 2^e < 1 (0 when all zero)
ENMF_DEV int exp_above(double mx) {
  if (!(mx > 0.0)) return 0;
  int e;
  frexp(mx, &e);            // mx = f · 2^e, f ∈ [0.5, 1)
  return e;
}

// X statistics once per load, in one pass each:
//  * row_stats: one block per row → e[i] (the row's exponent) and the max over rows of
//    max_k|x| / mean_k|x| (atomicMax on the positive ratio's bit pattern);
//  * col_stats_part: a 2-D grid of (column, row chunk) → per-chunk column max / sum;
//    col_stats_final: fixed-order chunk combine → e[k] and the ratio (deterministic).
__global__ void row_stats(const double* __restrict__ a, long K, long lda, int* e, unsigned long long* ratio_bits) {
  __shared__ double smax[32], ssum[32];
  const double* row = a + (long)blockIdx.x * lda;
  double m = 0.0, t = 0.0;
  for (long k = threadIdx.x; k < K; k += blockDim.x) {
    const double v = fabs(row[k]);
    m = fmax(m, v);
    t += v;
  }
  for (int o = 16; o; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  if ((threadIdx.x & 31) == 0) { smax[threadIdx.x >> 5] = m; ssum[threadIdx.x >> 5] = t; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0, tt = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { mm = fmax(mm, smax[w]); tt += ssum[w]; }
    e[blockIdx.x] = exp_above(mm);
    if (tt > 0.0) atomicMax(ratio_bits, (unsigned long long)__double_as_longlong(mm * (double)K / tt));
  }
}
__global__ void col_stats_part(const double* __restrict__ a, long R, long K, long lda, int chunks,
                               double* __restrict__ pmax, double* __restrict__ psum) {
  const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const long r0 = R * blockIdx.y / chunks, r1 = R * (blockIdx.y + 1) / chunks;
  double m = 0.0, t = 0.0;
  for (long i = r0; i < r1; ++i) {
    const double v = fabs(a[i * lda + k]);
    m = fmax(m, v);
    t += v;
  }
  pmax[(long)blockIdx.y * K + k] = m;
  psum[(long)blockIdx.y * K + k] = t;
}
__global__ void col_stats_final(const double* __restrict__ pmax, const double* __restrict__ psum, long R, long K,
                                int chunks, int* e, unsigned long long* ratio_bits) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (long)gridDim.x * blockDim.x) {
    double m = 0.0, t = 0.0;
    for (int c = 0; c < chunks; ++c) {
      m = fmax(m, pmax[(long)c * K + k]);
      t += psum[(long)c * K + k];
    }
    e[k] = exp_above(m);
    if (t > 0.0) atomicMax(ratio_bits, (unsigned long long)__double_as_longlong(m * (double)R / t));
  }
}

// digits of X once per load: row blockIdx.y, exponents per row (by_row) or per column;
// by_row also adds the row's digit sums into sums[p·R + i] (zeroed by the caller).  Eight
// consecutive elements per thread (K % 8 == 0, as the INT8 path requires 16-aligned shapes):
// four 16-byte loads, one 8-byte store per digit plane.
ENMF_DEV void split_x_row(const double* __restrict__ a, long i, long R, long K, long lda, const int* __restrict__ e,
                         int by_row, int8_t* __restrict__ out, int* __restrict__ sums) {
  const double* row = a + i * lda;
  int8_t* o = out + i * K;
  const long dstride = R * K;
  const int er = by_row ? e[i] : 0;
  int acc[SMAX] = {};
  for (long k = ((long)blockIdx.x * blockDim.x + threadIdx.x) * 8; k < K; k += (long)gridDim.x * blockDim.x * 8) {
    double v[8];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 t = *reinterpret_cast<const double2*>(row + k + 2 * h);
      v[2 * h] = t.x;
      v[2 * h + 1] = t.y;
    }
    unsigned long long packed[SMAX] = {};
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int ex = (by_row ? er : e[k + u]) + 1;
      int8_t dd[SMAX];
      int dig[SMAX];
      cut8(v[u] * __longlong_as_double((long long)(1023 - ex) << 52), dd, 1, dig);   // |z| < 1/2
#pragma unroll
      for (int p = 0; p < SMAX; ++p) {
        acc[p] += dig[p];
        packed[p] |= (unsigned long long)(unsigned char)dd[p] << (8 * u);
      }
    }
#pragma unroll
    for (int p = 0; p < SMAX; ++p) *reinterpret_cast<unsigned long long*>(o + p * dstride + k) = packed[p];
  }
  if (by_row) add_digit_sums(acc, sums + i, R);
}
// rows grid-strided over gridDim.y (≤ 65535)
__global__ void split_x(const double* __restrict__ a, long R, long K, long lda, const int* __restrict__ e, int by_row,
                        int8_t* __restrict__ out, int* __restrict__ sums) {
  for (long i = blockIdx.y; i < R; i += gridDim.y) split_x_row(a, i, R, K, lda, e, by_row, out, sums);
}

// column sums of the SMAX digit planes of an R × K int8 matrix: sums[p·K + k] (zeroed by the
// caller); grid (column blocks of 4 columns per thread, row chunks); K % 4 == 0
__global__ void digit_colsums(const int8_t* __restrict__ d, long R, long K, int chunks, int* __restrict__ sums) {
  const long k = ((long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k >= K) return;
  const long r0 = R * blockIdx.y / chunks, r1 = R * (blockIdx.y + 1) / chunks;
  int acc[SMAX][4] = {};
  for (long i = r0; i < r1; ++i)
#pragma unroll
    for (int p = 0; p < SMAX; ++p) {
      const char4 c = *reinterpret_cast<const char4*>(d + (long)p * R * K + i * K + k);
      acc[p][0] += c.x;
      acc[p][1] += c.y;
      acc[p][2] += c.z;
      acc[p][3] += c.w;
    }
#pragma unroll
  for (int p = 0; p < SMAX; ++p)
#pragma unroll
    for (int u = 0; u < 4; ++u) atomicAdd(sums + (long)p * K + k + u, acc[p][u]);
}

// Per-product factor path (R ≤ a few hundred rows, K long): row maxima with many blocks per
// row (bit patterns of non-negative doubles order like the values: atomicMax on them), then
// the digits in a 2-D grid (row = blockIdx.y, no divisions) that also derives the exponent.
__global__ void row_absmax(const double* __restrict__ a, long K, long lda, unsigned long long* mx,
                           const DevState* st) {
  if (st && !dev_active(st)) return;
  __shared__ double sh[32];
  const double* row = a + (long)blockIdx.y * lda;
  double m = 0.0;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(row[k]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    atomicMax(mx + blockIdx.y, (unsigned long long)__double_as_longlong(m));
  }
}

// digits of row blockIdx.y (SMAX planes, plane stride R·K) from its maximum; block (0, i)
// also publishes the row's exponent for the recombination
// (and adds the row's digit sums into sums[p·R + i], zeroed by the caller)
__global__ void split_rows(const double* __restrict__ a, long R, long K, long lda,
                           const unsigned long long* mx, int* e_out, int8_t* __restrict__ out,
                           int* __restrict__ sums, const DevState* st) {
  if (st && !dev_active(st)) return;
  const long i = blockIdx.y;
  const int e = exp_above(__longlong_as_double((long long)mx[i]));
  if (blockIdx.x == 0 && threadIdx.x == 0) e_out[i] = e;
  const double scale = __longlong_as_double((long long)(1023 - e - 1) << 52);   // 2^-(e+1), exact (|e| small)
  const double* row = a + i * lda;
  int8_t* o = out + i * K;
  const long dstride = R * K;
  int acc[SMAX] = {};
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (long)gridDim.x * blockDim.x) {
    int dig[SMAX];
    cut8(row[k] * scale, o + k, dstride, dig);     // |z| < 1/2
#pragma unroll
    for (int p = 0; p < SMAX; ++p) acc[p] += dig[p];
  }
  add_digit_sums(acc, sums + i, R);
}

// out[i][j] = sum_{q} sum_{p < S-q} 2^{ea_i + eb_j + 2 - 8(p+q+2)} · (D^A_p·D^B_q)_ij with
// D^A_p·D^B_q = Cq[p·R + i][j] + c_q·asum[p][i] + c_p·bsum[q][j] + c_p·c_q·K  (Cq = C + off.q[q],
// c_0 = 0, c_p = 128), exact in int64; FP64 sum smallest weight first.  out row stride ldo.
struct Offsets { long q[SMAX]; };   // start of digit GEMM q's output (its rows p·R + i, p < S - q)

// eb: the X digits' exponents, per output column j (X scaled per row for T·Xᵀ, per column for W_yᵀX)
// (two blocks per SM: more loads in flight for this memory-bound recombination; measured 2.50 ->
// 2.43 ms per C5 product including the digit GEMMs)
template <int S>
__global__ void __launch_bounds__(256, 2) combine(const int* __restrict__ C, Offsets off, long R, long N, long K, const int* ea, const int* eb,
                        const int* __restrict__ asum, const int* __restrict__ bsum, double* __restrict__ out, long ldo,
                        const DevState* st) {
  if (st && !dev_active(st)) return;
  const long i = blockIdx.y;
  const int ei = ea[i];
  int as[S];
#pragma unroll
  for (int p = 0; p < S; ++p) as[p] = asum[(long)p * R + i];
  for (long j = (long)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (long)gridDim.x * blockDim.x) {
    long long v[S][S];                               // v[q][p] = D^A_p·D^B_q, p + q < S
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const long long bs = 128LL * bsum[(long)q * N + j];   // c_p·colsum(d^B_q) for p ≥ 1
#pragma unroll
      for (int p = 0; p < S - q; ++p) {
        long long t = __ldcs(C + off.q[q] + ((long)p * R + i) * N + j);
        if (q) t += 128LL * as[p];                   // c_q·rowsum(d^A_p)
        if (p) t += bs;
        if (p && q) t += 16384LL * K;                // c_p·c_q·K
        v[q][p] = t;
      }
    }
    const int base = ei + eb[j] + 2;
    // The truncated part is not noise: the deep digits of real data are uniform in [0, 255], so
    // dropping the pairs p + q >= S and the uncut residuals biases every product low.  Its
    // expectation, from the digit sums along k (Σ_k D^A_p D^B_q ≈ Σ_k D^A_p · Σ_k D^B_q / K for
    // the dropped pairs; residuals uniform in [0, 256^-S)), is added first.
    double ra[S], cb[S];
#pragma unroll
    for (int p = 0; p < S; ++p) {
      ra[p] = (double)as[p] + (p ? 128.0 * (double)K : 0.0);
      cb[p] = (double)bsum[(long)p * N + j] + (p ? 128.0 * (double)K : 0.0);
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
    double acc = ldexp(corr, base);
#pragma unroll
    for (int w = S - 1; w >= 0; --w) {             // smallest weight 2^{-8(w+2)} first
      long long part = 0;                            // exact: at most S terms below 2^32 each
#pragma unroll
      for (int q = 0; q <= w; ++q) part += v[q][w - q];
      acc += ldexp((double)part, base - 8 * (w + 2));
    }
    out[i * ldo + j] = acc;
  }
}

}  // namespace ozaki

// ozaki.cuh — the digit scheme of the FP64-accurate cross products on the INT8 tensor cores
// (the cut, the per-row / per-column exponents and X's dynamic-range statistics); the digit
// layouts, the tcgen05 GEMM and the recombination are in ozk.cuh.
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
// each d^A_p·d^B_q an int8×int8→int32 tensor-core product (exact per K unit of ≤ 16384,
// ozk.cuh), the corrections exact integers.  With S = 6 levels (21 digit pairs) the neglected
// terms are ~2^{-47} of the row maxima — below FP64 accumulation over K = 32768 — and their
// expectation is added as a bias estimate (ozk::finish).  X's digits are cut once per load
// (X is fixed); the factor's digits once per product.
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

}  // namespace ozaki

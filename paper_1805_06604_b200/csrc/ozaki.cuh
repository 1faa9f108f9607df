// ozaki.cuh — FP64-accurate cross products on the B200's INT8 tensor cores.
//
// W_yᵀX and T·Xᵀ (linalg.hpp:67-124) are the two large contractions of an outer
// iteration (2·r·m·n flop each).  B200 runs FP64 on DMMA.8x8x4 at 37 TF/s but
// INT8 on tcgen05 at ~3 POP/s (profiles/r01_int8_probe.txt), so the products are
// computed by error-free splitting (Ozaki's scheme): every operand row is scaled
// by a power of two into (-1, 1) and cut into S signed 7-bit digits,
//     a = 2^e · sum_{p<S} d_p · 2^{-7(p+1)},   d_p ∈ [-127, 127]   (exact cuts)
// and the product is the exact int32 sum of the digit products
//     (A·B)_ij ≈ 2^{ea_i+eb} · sum_{p+q<S} 2^{-7(p+q+2)} · (D^A_p · D^B_q)_ij
// each digit GEMM an int8×int8→int32 tensor-core GEMM (exact while K·127² < 2³¹).
// With S = 7 the neglected terms are below 2^{-49} of the row maxima — the same
// order as FP64 accumulation over K = 32768 — and the sum over the digit pairs is
// formed in FP64 smallest term first.  X's digits are cut once per load (X is
// fixed); the factor's digits once per product.  The digit GEMMs are grouped by
// X digit q: one GEMM multiplies the stacked factor digits p = 0..S-1-q (an
// (S-q)·r-row operand) by X digit q, so X is streamed S times per product.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace ozaki {

constexpr int SMAX = 8;                   // digits cut per operand (7 bits each)
// digit levels kept, S ∈ {7, 8}: products d_p·d_q with p + q < S (S(S+1)/2 of them).  7 levels
// for X with a narrow per-row / per-column dynamic range, 8 otherwise (see ozaki_levels)

// largest |x| → exponent e with |x| / 2^e < 1 (0 when all zero)
ENMF_DEV int exp_above(double mx) {
  if (!(mx > 0.0)) return 0;
  int e;
  frexp(mx, &e);            // mx = f · 2^e, f ∈ [0.5, 1)
  return e;
}

__global__ void absmax_partial(const double* __restrict__ x, long cnt, double* part) {
  __shared__ double sh[32];
  double m = 0.0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) part[blockIdx.x] = m;
  }
}

__global__ void absmax_final(const double* part, int nb, int* e_out) {
  double m = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) m = fmax(m, part[i]);
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    m = fmax(m, sh[0]);
    *e_out = exp_above(m);
  }
}

// one block per row of an R × K row-major matrix: e[i] for max_k |a[i][k]|
__global__ void row_exp(const double* __restrict__ a, long K, long lda, int* e, const DevState* st) {
  if (st && !dev_active(st)) return;
  __shared__ double sh[32];
  const double* row = a + (long)blockIdx.x * lda;
  double m = 0.0;
  for (long k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, fabs(row[k]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    m = fmax(m, sh[0]);
    e[blockIdx.x] = exp_above(m);
  }
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

// digits of X once per load: row blockIdx.y, exponents per row (by_row) or per column
__global__ void split_x(const double* __restrict__ a, long R, long K, long lda, const int* __restrict__ e, int by_row,
                        int8_t* __restrict__ out) {
  const long i = blockIdx.y;
  const double* row = a + i * lda;
  int8_t* o = out + i * K;
  const long dstride = R * K;
  const int er = by_row ? e[i] : 0;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (long)gridDim.x * blockDim.x) {
    const int ex = by_row ? er : e[k];
    double r = row[k] * __longlong_as_double((long long)(1023 - ex) << 52);   // exact, |r| < 1
#pragma unroll
    for (int p = 0; p < SMAX; ++p) {
      r *= 128.0;
      const double d = trunc(r);
      r -= d;
      o[p * dstride + k] = (int8_t)(int)d;
    }
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

// digits of row blockIdx.y (SMAX planes, plane stride R·K) from its maximum; block (0, i)
// also publishes the row's exponent for the recombination
__global__ void split_rows(const double* __restrict__ a, long R, long K, long lda,
                           const unsigned long long* mx, int* e_out, int8_t* __restrict__ out,
                           const DevState* st) {
  if (st && !dev_active(st)) return;
  const long i = blockIdx.y;
  const int e = exp_above(__longlong_as_double((long long)mx[i]));
  if (blockIdx.x == 0 && threadIdx.x == 0) e_out[i] = e;
  const double scale = __longlong_as_double((long long)(1023 - e) << 52);   // 2^-e, exact (|e| small)
  const double* row = a + i * lda;
  int8_t* o = out + i * K;
  const long dstride = R * K;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (long)gridDim.x * blockDim.x) {
    double r = row[k] * scale;                      // exact, |r| < 1
#pragma unroll
    for (int p = 0; p < SMAX; ++p) {
      r *= 128.0;
      const double d = trunc(r);
      r -= d;
      o[p * dstride + k] = (int8_t)(int)d;
    }
  }
}

// e[k] for max_i |a[i][k]| of an R × K row-major matrix (thread per column, coalesced rows)
__global__ void col_exp(const double* __restrict__ a, long R, long K, long lda, int* e) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (long)gridDim.x * blockDim.x) {
    double m = 0.0;
    for (long i = 0; i < R; ++i) m = fmax(m, fabs(a[i * lda + k]));
    e[k] = exp_above(m);
  }
}

// Dynamic range of an R × K row-major matrix along K: ratio[0] = max over rows of
// max_k |a| / mean_k |a| (rows with a zero sum are skipped).  One block per row.
__global__ void row_range(const double* __restrict__ a, long K, long lda, unsigned long long* ratio_bits) {
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
    double tt = 0.0;
    m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      m = fmax(m, smax[w]);
      tt += ssum[w];
    }
    if (tt > 0.0) {
      const double ratio = m * (double)K / tt;      // positive: the bit pattern orders like the value
      atomicMax(ratio_bits, (unsigned long long)__double_as_longlong(ratio));
    }
  }
}
// Same along the rows: thread per column.
__global__ void col_range(const double* __restrict__ a, long R, long K, long lda, unsigned long long* ratio_bits) {
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += (long)gridDim.x * blockDim.x) {
    double m = 0.0, t = 0.0;
    for (long i = 0; i < R; ++i) {
      const double v = fabs(a[i * lda + k]);
      m = fmax(m, v);
      t += v;
    }
    if (t > 0.0) atomicMax(ratio_bits, (unsigned long long)__double_as_longlong(m * (double)R / t));
  }
}

// digits of an R × K matrix (row-major, lda) into out[p][i][k] (row stride K,
// digit stride R·K); row i is scaled by 2^-e[i] (per_row) or 2^-e[0].
// scale: 0 = one exponent e[0], 1 = per row e[i], 2 = per column e[k]; SMAX digits
__global__ void split(const double* __restrict__ a, long R, long K, long lda, const int* e, int scale,
                      int8_t* __restrict__ out, const DevState* st) {
  if (st && !dev_active(st)) return;
  const long total = R * K, dstride = R * K;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const long i = idx / K, k = idx - i * K;
    double r = ldexp(a[i * lda + k], -e[scale == 1 ? i : scale == 2 ? k : 0]);   // exact, |r| < 1
#pragma unroll
    for (int p = 0; p < SMAX; ++p) {
      r *= 128.0;                      // exact
      const double d = trunc(r);       // |d| <= 127
      r -= d;                          // exact
      out[p * dstride + idx] = (int8_t)(int)d;
    }
  }
}

// out[i][j] = sum_{q} sum_{p < S-q} 2^{ea_i + eb - 7(p+q+2)} · Cq[p·R + i][j],  Cq = C + off.q[q]
// (FP64, smallest weight first).  out row stride ldo.
struct Offsets { long q[SMAX]; };   // start of digit GEMM q's output (its rows p·R + i, p < S - q)

// eb: the X digits' exponents, per output column j (X scaled per row for T·Xᵀ, per column for W_yᵀX)
template <int S>
__global__ void combine(const int* __restrict__ C, Offsets off, long R, long N, const int* ea, const int* eb,
                        double* __restrict__ out, long ldo, const DevState* st) {
  if (st && !dev_active(st)) return;
  const long i = blockIdx.y;
  const int ei = ea[i];
  for (long j = (long)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (long)gridDim.x * blockDim.x) {
    int v[S][S];                                     // v[q][p] = digit product (p, q), p + q < S
#pragma unroll
    for (int q = 0; q < S; ++q)
#pragma unroll
      for (int p = 0; p < S - q; ++p) v[q][p] = __ldcs(C + off.q[q] + ((long)p * R + i) * N + j);
    const int base = ei + eb[j];
    double acc = 0.0;
#pragma unroll
    for (int w = S - 1; w >= 0; --w) {             // smallest weight 2^{-7(w+2)} first
      long long part = 0;                            // exact: at most S terms below 2^31 each
#pragma unroll
      for (int q = 0; q <= w; ++q) part += v[q][w - q];
      acc += ldexp((double)part, base - 7 * (w + 2));
    }
    out[i * ldo + j] = acc;
  }
}

}  // namespace ozaki

// sparse.cuh — the CSR cross products (linalg.hpp:86-104, 127-146) on sm_100a.
//
// X stays in the reference's CSR (row offsets + column indices + values) for
// X·Tᵀ and gets a CSC copy (built once at load, stable in the row order) for
// W_yᵀX, so both products are gathers without atomics:
//   (X·Tᵀ)[i][k] = sum_{p in row i} v_p · T[k][j_p]     warp per row,    lane per k
//   (W_yᵀX)[k][j] = sum_{p in col j} W_y[i_p][k] · v_p   warp per column, lane per k
// Each lane accumulates its element over the stored entries in the reference's
// order (rows ascending for a column, storage order within a row), so with
// EXACT (separately rounded multiply and add) the products are bitwise the
// reference's; the fast mode fuses them.  The gathered operand is kept row-major
// (T as n×r, W_y as m×r: one 8r-byte row per stored entry) — the engine
// transposes the r-major factors once per product.
// Bound: latency / L2 (nnz·(12 + 8r) bytes; the factors are L2-resident at C4).
#pragma once

#include "common.cuh"

namespace sparse {

// out[k·ldo + i] = sum_p v_p · G[idx_p·r + k] over the stored entries of line i
// (a CSR row or a CSC column); lines = rows (m) or columns (n).
template <bool EXACT>
__global__ void __launch_bounds__(256) gather_lines(const long long* ptr, const int* idx, const double* v,
                                                    const double* G, int lines, int r, double* out, long ldo,
                                                    const DevState* st) {
  if (st && !dev_active(st)) return;
  const int lane = threadIdx.x & 31;
  const long wid = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long i = wid; i < lines; i += nw) {
    const long p0 = ptr[i], p1 = ptr[i + 1];
    for (int k0 = 0; k0 < r; k0 += 32) {
      const int k = k0 + lane;
      double acc = 0.0;
      if (k < r) {
        for (long p = p0; p < p1; ++p) {
          const double x = __ldg(v + p);
          const double g = __ldg(G + (long)__ldg(idx + p) * r + k);
          acc = EXACT ? __dadd_rn(acc, __dmul_rn(g, x)) : fma(g, x, acc);
        }
        out[(long)k * ldo + i] = acc;
      }
    }
  }
}

// FP64 product mode, r <= 32: the stored entries of a line are dealt round-robin over the lanes
// (lane l takes entries l, l+32, …, each contributing its whole gathered row to r accumulators),
// then one reduce-scatter leaves the total for k = l in lane l.  The dependent chain per line
// drops from its length to length/32, which is what matters for the term rows of a Zipf corpus
// (the most frequent terms occur in most documents: one warp walking a 10^4-entry row was the
// whole X·Tᵀ time at C4).  Fixed order per line: deterministic.
// acc[k] += Σ_{p in [b, e), p ≡ b + lane (mod 32)} v_p · G[idx_p][k]  (k < r <= 32), then a
// reduce-scatter over the lanes: the returned value of lane l is the range's total for k = l.
ENMF_DEV double range_sum_lanes(long b, long e, const int* idx, const double* v, const double* G, int r, int lane) {
  double acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0;
  if ((r & 1) == 0) {
    // even r: the gathered row (8r bytes, 16-byte aligned) in 16-byte loads
    for (long p = b + lane; p < e; p += 32) {
      const double x = __ldg(v + p);
      const double2* g = reinterpret_cast<const double2*>(G + (long)__ldg(idx + p) * r);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (2 * k < r) {
          const double2 t = __ldg(g + k);
          acc[2 * k] = fma(t.x, x, acc[2 * k]);
          acc[2 * k + 1] = fma(t.y, x, acc[2 * k + 1]);
        }
    }
  } else {
    for (long p = b + lane; p < e; p += 32) {
      const double x = __ldg(v + p);
      const double* g = G + (long)__ldg(idx + p) * r;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (k < r) acc[k] = fma(__ldg(g + k), x, acc[k]);
    }
  }
  // reduce-scatter: afterwards acc[0] of lane l is the total for k = l
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool upper = (lane & w) != 0;
#pragma unroll
    for (int j = 0; j < w; ++j) {
      const double send = upper ? acc[j] : acc[j + w];
      const double keep = upper ? acc[j + w] : acc[j];
      acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return acc[0];
}

// FP64 product mode, r <= 32: the stored entries of a line are dealt round-robin over the lanes
// (lane l takes entries l, l+32, …, each contributing its whole gathered row to r accumulators),
// then one reduce-scatter leaves the total for k = l in lane l.  Fixed order: deterministic.
__global__ void __launch_bounds__(256) gather_lines_par(const long long* ptr, const int* idx, const double* v,
                                                        const double* G, int lines, int r, double* out, long ldo,
                                                        const DevState* st) {
  if (st && !dev_active(st)) return;
  const int lane = threadIdx.x & 31;
  const long wid = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long i = wid; i < lines; i += nw) {
    const double t = range_sum_lanes(ptr[i], ptr[i + 1], idx, v, G, r, lane);
    if (lane < r) out[(long)lane * ldo + i] = t;
  }
}

// Same, over fixed-size chunks of the lines (built once at load): the Zipf term rows of a
// document corpus (≈10⁴ entries for the most frequent terms) are split over many warps instead of
// walking one warp through them.  A single-chunk line is written directly; a split line's chunk
// totals go to part[slot·r + k] and combine_chunks adds them in chunk order (deterministic).
__global__ void __launch_bounds__(256) gather_chunks(const int* cline, const long long* cbeg, const long long* cend,
                                                     const int* cslot, int nchunks, const int* idx, const double* v,
                                                     const double* G, int r, double* out, long ldo, double* part,
                                                     const DevState* st) {
  if (st && !dev_active(st)) return;
  const int lane = threadIdx.x & 31;
  const long wid = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long c = wid; c < nchunks; c += nw) {
    const double t = range_sum_lanes(cbeg[c], cend[c], idx, v, G, r, lane);
    if (lane < r) {
      const int slot = cslot[c];
      if (slot < 0) out[(long)lane * ldo + cline[c]] = t;
      else part[(long)slot * r + lane] = t;
    }
  }
}

__global__ void combine_chunks(const int* mline, const int* mfirst, const int* mcount, int nmulti, const double* part,
                               int r, double* out, long ldo, const DevState* st) {
  if (st && !dev_active(st)) return;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < (long)nmulti * r; e += (long)gridDim.x * blockDim.x) {
    const int l = (int)(e / r), k = (int)(e % r);
    double t = 0.0;
    for (int q = 0; q < mcount[l]; ++q) t += part[(long)(mfirst[l] + q) * r + k];
    out[(long)k * ldo + mline[l]] = t;
  }
}

}  // namespace sparse

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

}  // namespace sparse

// bpp.cuh — batched exact NNLS by block principal pivoting (nnls.hpp:259-406).
//
// One warp per right-hand side (column).  The reference groups columns with
// identical passive sets to share one Cholesky factor; every per-column
// result (factor, pivot drops/bans, iterates, exchanges) is a function of the
// passive set alone, so per-column solving reproduces it exactly (SURVEY §3.4,
// verified column-by-column there).  Every reduction below keeps the
// reference's sequential order with separately rounded multiply/subtract, so
// given the same Gram and cross products a column's result is bitwise the
// reference's:
//   cholesky       nnls.hpp:215-229  (column j: pivot by lane 0, rows i>j lane-parallel,
//                                     each with its own sequential p-loop)
//   cholesky_solve nnls.hpp:232-243  (lane 0, sequential)
//   refinement     nnls.hpp:349-359  (rows lane-parallel, sequential b-loop)
//   feasibility    nnls.hpp:362-373  (lane-parallel, sequential a-loop)
//   exchange rules nnls.hpp:384-400  (full flip / backup(3) / largest index)
// Passive/banned/infeasible sets are bit masks of RM/64 64-bit words (Bits<W>), r <= RM <= 128;
// at RM = 128 the per-warp factor is stored packed lower-triangular so G and L fit the
// shared memory of one warp per block.
#pragma once

#include "common.cuh"
#include "dist.cuh"

namespace bpp {

constexpr int MAXR = 128;

// fixed-size bit set over r <= 64·W indices
template <int W>
struct Bits {
  unsigned long long w[W];
  ENMF_DEV void clear() {
#pragma unroll
    for (int i = 0; i < W; ++i) w[i] = 0;
  }
  ENMF_DEV bool test(int i) const { return (w[i >> 6] >> (i & 63)) & 1ULL; }
  ENMF_DEV void set(int i) { w[i >> 6] |= 1ULL << (i & 63); }
  ENMF_DEV void reset(int i) { w[i >> 6] &= ~(1ULL << (i & 63)); }
  ENMF_DEV void flip(int i) { w[i >> 6] ^= 1ULL << (i & 63); }
  ENMF_DEV void xor_with(const Bits& o) {
#pragma unroll
    for (int i = 0; i < W; ++i) w[i] ^= o.w[i];
  }
  ENMF_DEV bool any() const {
    unsigned long long v = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) v |= w[i];
    return v != 0;
  }
  ENMF_DEV int count() const {
    int c = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) c += __popcll(w[i]);
    return c;
  }
  ENMF_DEV int highest() const {   // largest set index (any() must hold)
#pragma unroll
    for (int i = W - 1; i >= 0; --i)
      if (w[i]) return 64 * i + 63 - __clzll(w[i]);
    return -1;
  }
};

struct Args {
  const double* G;        // r×r
  const double* C;        // r×N, row stride ld
  const double* H0;       // warm start r×N
  double* H;              // solution r×N
  long ld;
  int r, N;
  const double* cmax;     // max |C| (device scalar)
  DevState* st;           // nullable
  int side;
  unsigned long long* exchanges;  // total exchanges (atomic)
  int* rounds;                    // max solves per column (atomic max)
  int* nonfinite;                 // set if a non-finite value is written
};

template <int RM>
__host__ __device__ constexpr int l_elems() { return RM <= 64 ? RM * (RM + 1) : RM * (RM + 1) / 2; }   // L storage per warp

template <int RM, int WPB>
constexpr int smem_bytes() {
  // G (RM×(RM+1), odd row stride) + per warp: L (RM×(RM+1): the odd row stride keeps the
  // lane-per-row loads of the factorization off one bank; packed triangle at RM = 128),
  // x/d/res (3×RM), fidx (RM ints)
  return RM * (RM + 1) * 8 + WPB * (l_elems<RM>() * 8 + 3 * RM * 8 + RM * 4);
}

ENMF_DEV unsigned long long warp_or64(unsigned long long v) {
  const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)(v & 0xffffffffULL));
  const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(v >> 32));
  return ((unsigned long long)hi << 32) | lo;
}
template <int W>
ENMF_DEV Bits<W> warp_or(Bits<W> b) {
#pragma unroll
  for (int i = 0; i < W; ++i) b.w[i] = warp_or64(b.w[i]);
  return b;
}
template <int W>
ENMF_DEV Bits<W> shfl0(Bits<W> b) {
#pragma unroll
  for (int i = 0; i < W; ++i) b.w[i] = __shfl_sync(0xffffffffu, b.w[i], 0);
  return b;
}

template <int RM, int WPB>
__global__ void __launch_bounds__(WPB * 32) solve(Args a) {
  if (a.st && !dev_active(a.st)) return;
  extern __shared__ __align__(16) double sm[];
  const int r = a.r;
  double* Gs = sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int W = (RM + 63) / 64;
  constexpr int LDL = RM + 1;             // row stride of L (bank spread for lane-per-row access)
  constexpr int LE = l_elems<RM>();
  // L(i, p), p <= i: strided rows, or the packed lower triangle at RM = 128
  auto LI = [](int i, int p) { return RM <= 64 ? i * LDL + p : i * (i + 1) / 2 + p; };
  double* L = sm + RM * LDL + warp * (LE + 3 * RM);
  double* xf = L + LE;
  double* df = xf + RM;
  double* rs = df + RM;
  int* fidx = reinterpret_cast<int*>(sm + RM * LDL + WPB * (LE + 3 * RM)) + warp * RM;

  const int gld = r | 1;                   // odd row stride of the Gram copy (bank spread)
  for (int e = threadIdx.x; e < r * r; e += WPB * 32) Gs[(e / r) * gld + e % r] = a.G[e];
  __syncthreads();

  double maxd = 0.0;
  for (int i = 0; i < r; ++i) maxd = (maxd < Gs[i * gld + i]) ? Gs[i * gld + i] : maxd;
  const double pivot_floor = __dmul_rn(1e-12, maxd);
  const double feas_tol = __dmul_rn(1e-12, __dadd_rn(1.0, *a.cmax));
  const unsigned long long limit = 3ULL * (unsigned long long)r * (unsigned long long)a.N;

  for (int col = blockIdx.x * WPB + warp; col < a.N; col += gridDim.x * WPB) {
    Bits<W> P, B;
    P.clear();
    B.clear();
    for (int i = lane; i < r; i += 32)
      if (a.H0[(long)i * a.ld + col] > 0.0) P.set(i);
    P = warp_or(P);
    int best_inf = 0x7fffffff, backup = 3, solves = 0;
    unsigned long long exch = 0;
    int f = 0;
    for (;;) {
      ++solves;
      // passive index list (ascending)
      f = 0;
      if (lane == 0)
        for (int i = 0; i < r; ++i)
          if (P.test(i)) fidx[f++] = i;
      f = __shfl_sync(0xffffffffu, f, 0);
      __syncwarp();
      // factor G[F,F], dropping and banning variables whose pivot collapses
      for (;;) {
        if (f == 0) break;
        int bad = f;
        for (int j = 0; j < f; ++j) {
          double ljj = 0.0;
          int ok = 1;
          if (lane == 0) {
            double d = Gs[fidx[j] * gld + fidx[j]];
            for (int p = 0; p < j; ++p) d = __dsub_rn(d, __dmul_rn(L[LI(j, p)], L[LI(j, p)]));
            ok = (d > pivot_floor) ? 1 : 0;
            if (ok) {
              ljj = __dsqrt_rn(d);
              L[LI(j, j)] = ljj;
            }
          }
          ok = __shfl_sync(0xffffffffu, ok, 0);
          if (!ok) { bad = j; break; }
          ljj = __shfl_sync(0xffffffffu, ljj, 0);
          __syncwarp();
          for (int i = j + 1 + lane; i < f; i += 32) {
            double s = Gs[fidx[i] * gld + fidx[j]];
            for (int p = 0; p < j; ++p) s = __dsub_rn(s, __dmul_rn(L[LI(i, p)], L[LI(j, p)]));
            L[LI(i, j)] = __ddiv_rn(s, ljj);
          }
          __syncwarp();
        }
        if (bad == f) break;
        if (lane == 0) {
          const int var = fidx[bad];
          P.reset(var);
          B.set(var);
          for (int q = bad; q + 1 < f; ++q) fidx[q] = fidx[q + 1];
        }
        P = shfl0(P);
        B = shfl0(B);
        --f;
        __syncwarp();
      }
      // x_F = chol_solve(C[F,col]) + one refinement step
      for (int q = lane; q < f; q += 32) df[q] = a.C[(long)fidx[q] * a.ld + col];
      __syncwarp();
      auto chol_solve = [&](double* b) {
        if (lane == 0) {
          for (int i = 0; i < f; ++i) {
            double s = b[i];
            for (int p = 0; p < i; ++p) s = __dsub_rn(s, __dmul_rn(L[LI(i, p)], b[p]));
            b[i] = __ddiv_rn(s, L[LI(i, i)]);
          }
          for (int ii = f - 1; ii >= 0; --ii) {
            double s = b[ii];
            for (int p = ii + 1; p < f; ++p) s = __dsub_rn(s, __dmul_rn(L[LI(p, ii)], b[p]));
            b[ii] = __ddiv_rn(s, L[LI(ii, ii)]);
          }
        }
        __syncwarp();
      };
      if (f > 0) {
        for (int q = lane; q < f; q += 32) xf[q] = df[q];
        __syncwarp();
        chol_solve(xf);
        for (int q = lane; q < f; q += 32) {
          double s = df[q];
          for (int b2 = 0; b2 < f; ++b2) s = __dsub_rn(s, __dmul_rn(Gs[fidx[q] * gld + fidx[b2]], xf[b2]));
          rs[q] = s;
        }
        __syncwarp();
        chol_solve(rs);
        for (int q = lane; q < f; q += 32) xf[q] = __dadd_rn(xf[q], rs[q]);
        __syncwarp();
      }
      // infeasible set
      Bits<W> I;
      I.clear();
      for (int q = lane; q < f; q += 32)
        if (xf[q] < -feas_tol) I.set(fidx[q]);
      for (int i = lane; i < r; i += 32) {
        if (P.test(i) || B.test(i)) continue;
        double y = -a.C[(long)i * a.ld + col];
        for (int q = 0; q < f; ++q) y = __dadd_rn(y, __dmul_rn(Gs[i * gld + fidx[q]], xf[q]));
        if (y < -feas_tol) I.set(i);
      }
      I = warp_or(I);
      if (!I.any()) break;
      if (++exch > limit) break;  // the total exceeds the global limit too
      const int count = I.count();
      if (count < best_inf) {
        best_inf = count;
        backup = 3;
        P.xor_with(I);
      } else if (backup > 0) {
        --backup;
        P.xor_with(I);
      } else {
        P.flip(I.highest());
      }
    }
    // write the column: max(x, 0) on F, zero elsewhere
    int nf = 0;
    for (int i = lane; i < r; i += 32) a.H[(long)i * a.ld + col] = 0.0;
    __syncwarp();
    for (int q = lane; q < f; q += 32) {
      const double v = xf[q] > 0.0 ? xf[q] : 0.0;
      a.H[(long)fidx[q] * a.ld + col] = v;
      nf |= !isfinite(v);
    }
    nf = __any_sync(0xffffffffu, nf);
    if (lane == 0) {
      if (exch) atomicAdd(a.exchanges, exch);
      atomicMax(a.rounds, solves);
      if (nf) atomicOr(a.nonfinite, 1);
    }
    __syncwarp();
  }
}


// ---- lane-parallel solver (FP64 product mode, r <= 32) -------------------------------
//
// Same block-principal-pivoting control flow as `solve` (passive-set exchanges, pivot
// drop/ban, one refinement step, full / backup(3) / largest-index rules, nnls.hpp:259-406),
// but the arithmetic is spread over the warp instead of following the reference's sequential
// order: lane q owns row q of the passive set; the Cholesky factor of G[F,F] is formed
// right-looking (per pivot: one broadcast, a lane-parallel scale and a lane-parallel trailing
// update), the triangular solves are lane-parallel column sweeps with the pivot reciprocals
// precomputed, FMA throughout.  The dependent chain per round shrinks from O(f²) serial
// FP64 ops on lane 0 to O(f); the result is the same NNLS solution up to rounding (the
// bitwise-faithful `solve` stays the kernel of `fp64_exact` and of the kernel-level API).
template <int WPB>
constexpr int fast_smem_bytes() {
  // G (32×33) + per warp: L (32×33), x (32), 1/diag (32), fidx (32 ints); + the lower-triangle
  // index table (528 packed (u, v) pairs) shared by the block
  return 32 * 33 * 8 + WPB * (32 * 33 * 8 + 2 * 32 * 8 + 32 * 4) + 528 * 4;
}

// One column of the lane-parallel solver (FP64 product mode, r <= 32): warp-collective.
// Gs: the Gram in shared memory (row stride gld); tri: the lower-triangle index table; L (32 ×
// LDL), xs, invd (32 each), fidx (32 ints): this warp's shared-memory workspace.  C, H0 (read)
// and H (written) are r × N with row stride ld.  Returns the solve count; *exch / *nf get the
// column's exchanges and non-finite flag.
struct FastCol {
  const double* Gs;
  int gld;
  const int* tri;
  double* L;
  double* xs;
  double* invd;
  int* fidx;
  int r;
  double pivot_floor, feas_tol;
  unsigned long long limit;
};
ENMF_DEV int solve_fast_col(const FastCol& w, const double* C, const double* H0, double* H, long ld, long col,
                            unsigned long long* exch_out, int* nf_out) {
  constexpr int LDL = 33;
  const int lane = threadIdx.x & 31;
  const int r = w.r, gld = w.gld;
  const double* Gs = w.Gs;
  const int* tri = w.tri;
  double* L = w.L;
  double* xs = w.xs;
  double* invd = w.invd;
  int* fidx = w.fidx;
  // lane-parallel triangular solves with the factor in L: b (lane q's entry) -> A⁻¹ b
  auto chol_solve = [&](double b, int f) -> double {
    for (int i = 0; i < f; ++i) {                 // forward: L y = b
      const double yi = __shfl_sync(0xffffffffu, b, i) * invd[i];
      if (lane == i) b = yi;
      else if (lane > i && lane < f) b = fma(-L[lane * LDL + i], yi, b);
    }
    for (int i = f - 1; i >= 0; --i) {            // backward: Lᵀ x = y
      const double xi = __shfl_sync(0xffffffffu, b, i) * invd[i];
      if (lane == i) b = xi;
      else if (lane < i) b = fma(-L[i * LDL + lane], xi, b);
    }
    return b;
  };
  unsigned long long P = 0, B = 0;
  if (lane < r && H0[(long)lane * ld + col] > 0.0) P = 1ULL << lane;
  P = warp_or64(P);
  int best_inf = 0x7fffffff, backup = 3, solves = 0;
  unsigned long long exch = 0;
  int f = 0, fq = 0;
  double x = 0.0;                               // lane q: x_F[q]
  for (;;) {
    ++solves;
    // passive index list (ascending) from the mask
    const unsigned pm = (unsigned)P;
    if (lane < r && ((pm >> lane) & 1u)) fidx[__popc(pm & ((1u << lane) - 1u))] = lane;
    f = __popc(pm);
    __syncwarp();
    // factor G[F,F] right-looking, dropping and banning variables whose pivot collapses
    for (;;) {
      if (f == 0) break;
      fq = lane < f ? fidx[lane] : 0;
      if (lane < f)
        for (int k = 0; k <= lane; ++k) L[lane * LDL + k] = Gs[fq * gld + fidx[k]];
      __syncwarp();
      int bad = f;
      for (int j = 0; j < f; ++j) {
        const double d = L[j * LDL + j];
        if (!(d > w.pivot_floor)) { bad = j; break; }
        const double ljj = sqrt(d), inv = 1.0 / ljj;
        if (lane > j && lane < f) L[lane * LDL + j] = L[lane * LDL + j] * inv;
        if (lane == j) {
          L[j * LDL + j] = ljj;
          invd[j] = inv;
        }
        __syncwarp();
        // trailing update L[i][k] -= L[i][j]·L[k][j] (j < k <= i < f), the triangle's entries
        // dealt round-robin over the lanes (balanced, instead of one row per lane)
        const int nt = f - j - 1;
        for (int e = lane; e < nt * (nt + 1) / 2; e += 32) {
          const int uv = tri[e], i = j + 1 + (uv >> 8), k = j + 1 + (uv & 255);
          L[i * LDL + k] = fma(-L[i * LDL + j], L[k * LDL + j], L[i * LDL + k]);
        }
        __syncwarp();
      }
      if (bad == f) break;
      if (lane == 0) {
        const int var = fidx[bad];
        P &= ~(1ULL << var);
        B |= 1ULL << var;
        for (int q = bad; q + 1 < f; ++q) fidx[q] = fidx[q + 1];
      }
      P = __shfl_sync(0xffffffffu, P, 0);
      B = __shfl_sync(0xffffffffu, B, 0);
      --f;
      __syncwarp();
    }
    fq = lane < f ? fidx[lane] : 0;
    // x_F = chol_solve(C[F,col]) + one refinement step
    x = 0.0;
    if (f > 0) {
      const double df = lane < f ? C[(long)fq * ld + col] : 0.0;
      x = chol_solve(df, f);
      xs[lane] = x;
      __syncwarp();
      double rs = df;
      if (lane < f)
        for (int b2 = 0; b2 < f; ++b2) rs = fma(-Gs[fq * gld + fidx[b2]], xs[b2], rs);
      rs = chol_solve(rs, f);
      x += rs;
      __syncwarp();
      xs[lane] = x;
      __syncwarp();
    }
    // infeasible set
    unsigned long long I = 0;
    if (lane < f && x < -w.feas_tol) I = 1ULL << fq;
    if (lane < r && !(((P | B) >> lane) & 1ULL)) {
      double y = -C[(long)lane * ld + col];
      for (int q = 0; q < f; ++q) y = fma(Gs[lane * gld + fidx[q]], xs[q], y);
      if (y < -w.feas_tol) I |= 1ULL << lane;
    }
    I = warp_or64(I);
    if (I == 0) break;
    if (++exch > w.limit) break;
    const int count = __popcll(I);
    if (count < best_inf) {
      best_inf = count;
      backup = 3;
      P ^= I;
    } else if (backup > 0) {
      --backup;
      P ^= I;
    } else {
      P ^= 1ULL << (63 - __clzll(I));
    }
    __syncwarp();
  }
  // write the column: max(x, 0) on F, zero elsewhere
  int nf = 0;
  if (lane < r) H[(long)lane * ld + col] = 0.0;
  __syncwarp();
  if (lane < f) {
    const double v = x > 0.0 ? x : 0.0;
    H[(long)fq * ld + col] = v;
    nf = !isfinite(v);
  }
  *nf_out = __any_sync(0xffffffffu, nf);
  *exch_out = exch;
  __syncwarp();
  return solves;
}

// the index table of solve_fast_col's balanced trailing update: tri[u(u+1)/2 + v] = (u, v), v <= u < 32
ENMF_DEV void fill_tri(int* tri, int nwarps) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int u = warp; u < 32; u += nwarps)
    for (int v = lane; v <= u; v += 32) tri[u * (u + 1) / 2 + v] = (u << 8) | v;
}

template <int WPB>
__global__ void __launch_bounds__(WPB * 32) solve_fast(Args a) {
  if (a.st && !dev_active(a.st)) return;
  constexpr int LDL = 33;
  extern __shared__ __align__(16) double sm[];
  const int r = a.r;
  double* Gs = sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  FastCol w;
  w.L = sm + 32 * LDL + warp * (32 * LDL + 64);
  w.xs = w.L + 32 * LDL;
  w.invd = w.xs + 32;
  w.fidx = reinterpret_cast<int*>(sm + 32 * LDL + WPB * (32 * LDL + 64)) + warp * 32;
  int* tri = reinterpret_cast<int*>(sm + 32 * LDL + WPB * (32 * LDL + 64)) + WPB * 32;
  const int gld = r | 1;
  for (int e = threadIdx.x; e < r * r; e += WPB * 32) Gs[(e / r) * gld + e % r] = a.G[e];
  fill_tri(tri, WPB);
  __syncthreads();
  double maxd = 0.0;
  for (int i = 0; i < r; ++i) maxd = (maxd < Gs[i * gld + i]) ? Gs[i * gld + i] : maxd;
  w.Gs = Gs;
  w.gld = gld;
  w.tri = tri;
  w.r = r;
  w.pivot_floor = __dmul_rn(1e-12, maxd);
  w.feas_tol = __dmul_rn(1e-12, __dadd_rn(1.0, *a.cmax));
  w.limit = 3ULL * (unsigned long long)r * (unsigned long long)a.N;
  for (int col = blockIdx.x * WPB + warp; col < a.N; col += gridDim.x * WPB) {
    unsigned long long exch;
    int nf;
    const int solves = solve_fast_col(w, a.C, a.H0, a.H, a.ld, col, &exch, &nf);
    if (lane == 0) {
      if (exch) atomicAdd(a.exchanges, exch);
      atomicMax(a.rounds, solves);
      if (nf) atomicOr(a.nonfinite, 1);
    }
    __syncwarp();
  }
}

// Post-solve checks: exchange limit (NoConvergence, nnls.hpp:384-387) and the
// NaN guard on the solution (engine.hpp:334-337 / 380-383).
__global__ void check(DevState* st, int side, int r, int N, unsigned long long* exchanges, int* rounds,
                      int* nonfinite) {
  if (!st || !dev_active(st)) return;
  st->bpp_rounds[side] = *rounds;
  st->bpp_exchanges[side] = *exchanges;
  if (*exchanges > 3ULL * (unsigned long long)r * (unsigned long long)N) {
    st->error_code = ENMF_NO_CONVERGENCE;
    st->active = 0;
  } else if (*nonfinite) {
    st->error_code = ENMF_NON_FINITE;
    st->active = 0;
  }
  *exchanges = 0;
  *rounds = 0;
  *nonfinite = 0;
}

// max |C| over r×N (feas_tol, nnls.hpp:271).  Single block, order-independent.
__global__ void absmax(const double* C, long ld, int r, int N, double* out, const DevState* st,
                       const dist::View* dv = nullptr) {
  if (st && !dev_active(st)) return;
  __shared__ double red[256];
  double m = 0.0;
  for (long e = threadIdx.x; e < (long)r * N; e += blockDim.x) {
    const double v = fabs(C[(e / N) * ld + e % N]);
    m = (m < v) ? v : m;
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = dv ? dist::allmax_scalar(*dv, red[0]) : red[0];
}

}  // namespace bpp

// batch.cuh — packed many-small-runs backend: one CTA runs a WHOLE E-A-HALS / A-HALS / E-ANLS run
// (enmf::run, engine.hpp:447-521, every step() of it, engine.hpp:309-440) for one small dense
// problem, and one launch runs a batch of them (the paper protocol's dataset × init × algorithm
// grid, bench.hpp:233-294, which the reference spreads over host threads).
//
// A C1-class run (200 × 200, r = 20, 200 outer iterations) is ~57 graph nodes per iteration
// on the single-run engine, latency-bound at ~167 µs per iteration; here an iteration is a
// sequence of CTA-local phases separated by __syncthreads, with the problem's factors in L2 /
// shared memory and no launch, graph or host round trip between them:
//
//   gram(W_y) [+ reinit]      warp per Gram entry over the factor staged in shared memory
//   C_H = W_yᵀX               thread per column of X, r accumulators in registers
//   H update                  hals_solve, thread per column (r rows in registers, Gram in
//                             shared memory), fixed-order block reduction of the sweep gain
//   (hp ≥ 2) H_y              extrapolate (+ clamp for hp 3)
//   gram(T) [+ reinit], T·Xᵀ  warp per row of X, lanes over its columns, shuffle reduction
//   W update                  hals_solve on Wᵀ (thread per row of W)
//   W_y, (hp 1) H_y           extrapolate
//   error                     fast_error in double-double (||X||², ⟨W_n, X Tᵀ⟩, ⟨W_nᵀW_n, T Tᵀ⟩)
//   decide                    NaN guard, restart / accept, update_beta, IterationRecord
//
//   (E-ANLS) H / W update     active_set_solve by the engine's lane-parallel BPP column solver
//                             (bpp::solve_fast_col), six warps, a column per warp at a time
//
// Arithmetic is the engine's FP64 product mode (FMA, parallel reduction orders): parity with
// the reference is the north_star bar (identical restarts, errors within 1e-9, factors within
// 1e-6; tests/test_gpu_batch.py), not bit equality — the bitwise fp64_exact mode runs on the
// per-run engine (run_batch streams).  Limits: r ≤ 32, max(m, n)·⌈r⌉₈ ≤
// SMEM_FACTOR doubles (the staged factor), no wall-clock budget.
#pragma once

#include "bpp.cuh"
#include "common.cuh"

namespace batch {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int RMAX = 32;
constexpr int SMEM_FACTOR = 9216;      // doubles of the staged factor, max(m, n) × R (72 KB: two CTAs per SM)

struct Args {
  const double* x;          // count × m × n (row-major per run)
  const double* w0;         // count × m × r
  const double* h0;         // count × r × n
  double* w_out;            // count × m × r
  double* h_out;            // count × r × n
  enmf_gpu_iter* recs;      // count × cap
  int* n_recs;              // count
  int* status;              // count: ENMF_* of the run
  double* norm_x;           // count
  double* ws;               // gridDim.x × per-CTA workspace
  long count;
  int m, n, r;
  int cap;                  // record slots per run
  enmf_gpu_config cfg;
  int ms_h, ms_w;           // max sweeps per inner solve
};

// per-CTA workspace (doubles): WT, WyT, WnT, P (r × m); H, Hy, Hn, CH (r × n); scratch
__host__ __device__ inline long ws_doubles(int m, int n, int r) { return 4L * r * m + 4L * r * n + 64; }

// ---- block reductions (fixed order: deterministic) ----------------------------------
ENMF_DEV void dd_two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// (hi, lo) summed over the block; every thread gets the result
ENMF_DEV void block_dd_sum(double& hi, double& lo, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double oh = __shfl_xor_sync(0xffffffffu, hi, off), ol = __shfl_xor_sync(0xffffffffu, lo, off);
    double s, e;
    dd_two_sum(hi, oh, s, e);
    hi = s;
    lo = lo + ol + e;
  }
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    red[2 * w] = hi;
    red[2 * w + 1] = lo;
  }
  __syncthreads();
  hi = red[0];
  lo = red[1];
  for (int i = 1; i < NW; ++i) {
    double s, e;
    dd_two_sum(hi, red[2 * i], s, e);
    hi = s;
    lo = lo + red[2 * i + 1] + e;
  }
  __syncthreads();
}
ENMF_DEV double block_sum(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = red[0];
  for (int i = 1; i < NW; ++i) s += red[i];
  __syncthreads();
  return s;
}

// ---- factor phases (R: the rank rounded up to a multiple of 8, a compile-time constant;
// staged factors are [row][R] in shared memory, zero past r, so every inner loop is a fixed
// unrolled sequence of 16-byte broadcast loads and FMAs) ----------------------------------

// S (K × R, shared) = Aᵀ for A (r × K, global, row-major), zero-padded past r
template <int R>
ENMF_DEV void stage_t(const double* A, int r, int K, double* S) {
  for (int e = threadIdx.x; e < K * R; e += NT) {
    const int i = e / R, k = e % R;
    S[e] = k < r ? A[(long)k * K + i] : 0.0;
  }
}

// G (R × R, shared) = Sᵀ S for S (K × R, shared): thread per upper-triangle entry; padding rows /
// columns of G are zero
template <int R>
ENMF_DEV void gram_t(const double* S, int K, double* G) {
  constexpr int NP = R * (R + 1) / 2;
  for (int e = threadIdx.x; e < NP; e += NT) {
    int a = 0, rem = e;
    while (rem >= R - a) {
      rem -= R - a;
      ++a;
    }
    const int b = a + rem;
    double s0 = 0.0, s1 = 0.0;
    int i = 0;
    for (; i + 1 < K; i += 2) {
      s0 = fma(S[i * R + a], S[i * R + b], s0);
      s1 = fma(S[(i + 1) * R + a], S[(i + 1) * R + b], s1);
    }
    if (i < K) s0 = fma(S[i * R + a], S[i * R + b], s0);
    const double v = s0 + s1;
    G[a * R + b] = v;
    G[b * R + a] = v;
  }
  __syncthreads();
}

// gram_with_reinit (engine.hpp:268-296): degenerate rows of the factor (global Ag, r × K) are
// redrawn from mt19937_64(mix_seed(seed, salt, attempt)), restaged and the Gram recomputed.
// Returns 0 or ENMF_NO_CONVERGENCE; sets *modified.
template <int R>
ENMF_DEV int gram_reinit(double* Ag, double* S, int r, int K, double* G, uint64_t seed, uint64_t salt, int* modified,
                         int* sh_bad, int* sh_nb) {
  for (uint64_t attempt = 0;; ++attempt) {
    gram_t<R>(S, K, G);
    if (threadIdx.x == 0) {
      double maxd = 0.0;
      for (int i = 0; i < r; ++i) maxd = (maxd < G[i * R + i]) ? G[i * R + i] : maxd;
      const double fl = 1e-16 * maxd;
      int nb = 0;
      for (int k = 0; k < r; ++k)
        if (!(G[k * R + k] > fl)) sh_bad[nb++] = k;
      *sh_nb = nb;
    }
    __syncthreads();
    const int nb = *sh_nb;
    __syncthreads();
    if (nb == 0) return 0;
    if (attempt > (uint64_t)r + 2) return ENMF_NO_CONVERGENCE;
    if (threadIdx.x == 0) {
      DevMt64 gen;
      mt64_seed(gen, mix_seed(seed, salt, attempt));
      for (int q = 0; q < nb; ++q)
        for (int i = 0; i < K; ++i) {
          const double v = uniform_unit(gen);
          S[i * R + sh_bad[q]] = v;
          Ag[(long)sh_bad[q] * K + i] = v;
        }
      *modified = 1;
    }
    __syncthreads();
  }
}

// C (r × n, global) = Aᵀ X with A staged as S (m × R): thread per column j of X.
template <int R>
ENMF_DEV void cross_wx(const double* S, const double* X, int m, int n, int r, double* C) {
  for (int j = threadIdx.x; j < n; j += NT) {
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    const double* xc = X + j;
#pragma unroll 2
    for (int i = 0; i < m; ++i) {
      const double xv = __ldg(xc + (long)i * n);
      const double2* sr = reinterpret_cast<const double2*>(S + i * R);
#pragma unroll
      for (int k2 = 0; k2 < R / 2; ++k2) {
        const double2 w = sr[k2];
        acc[2 * k2] = fma(w.x, xv, acc[2 * k2]);
        acc[2 * k2 + 1] = fma(w.y, xv, acc[2 * k2 + 1]);
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (k < r) C[(long)k * n + j] = acc[k];
  }
}

// P (r × m, global) = T Xᵀ with T staged as S (n × R): thread per row i of X (the row is
// streamed through L1; all threads read the same S row: broadcast).
template <int R>
ENMF_DEV void cross_txt(const double* S, const double* X, int m, int n, int r, double* P) {
  for (int i = threadIdx.x; i < m; i += NT) {
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    const double* xr = X + (long)i * n;
#pragma unroll 2
    for (int j = 0; j < n; ++j) {
      const double xv = xr[j];
      const double2* sr = reinterpret_cast<const double2*>(S + j * R);
#pragma unroll
      for (int k2 = 0; k2 < R / 2; ++k2) {
        const double2 t = sr[k2];
        acc[2 * k2] = fma(t.x, xv, acc[2 * k2]);
        acc[2 * k2 + 1] = fma(t.y, xv, acc[2 * k2 + 1]);
      }
    }
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (k < r) P[(long)k * m + i] = acc[k];
  }
}

// Gauss-Seidel data from a Gram G (R × R, shared): Gz = G with a zero diagonal and zero padding,
// dinv = 1 / G_kk, dh = G_kk / 2 (padding rows: 1, 1/2)
template <int R>
ENMF_DEV void hals_prep(const double* G, int r, double* Gz, double* dinv) {
  for (int e = threadIdx.x; e < R * R; e += NT) {
    const int k = e / R, j = e % R;
    Gz[e] = (k == j || k >= r || j >= r) ? 0.0 : G[e];
  }
  for (int k = threadIdx.x; k < R; k += NT) dinv[k] = k < r ? 1.0 / G[k * R + k] : 1.0;
  __syncthreads();
}

// hals_solve (nnls.hpp:154-176) on r × N columns: warm start H0, output Hn (both r × N, global),
// C (r × N, global), Gz / dinv from hals_prep, G for the diagonal.  Thread per column, R values
// in registers.  Returns the sweep count; *nf |= a non-finite output.
template <int R>
ENMF_DEV int hals(const double* G, const double* Gz, const double* dinv, const double* C, const double* H0, double* Hn,
                  int r, int N, int max_sweeps, double stall, double* red, int* nf) {
  double first = 0.0;
  int sweep = 0;
  int bad = 0;
  for (;;) {
    ++sweep;
    double gain = 0.0;
    for (int t = threadIdx.x; t < N; t += NT) {
      double h[R];
      const double* src = sweep == 1 ? H0 : Hn;
#pragma unroll
      for (int k = 0; k < R; ++k) h[k] = k < r ? src[(long)k * N + t] : 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (k < r) {
          const double2* gk = reinterpret_cast<const double2*>(Gz + k * R);
          double s0 = C[(long)k * N + t], s1 = 0.0;
#pragma unroll
          for (int j2 = 0; j2 < R / 2; ++j2) {
            const double2 g = gk[j2];
            s0 = fma(-g.x, h[2 * j2], s0);
            s1 = fma(-g.y, h[2 * j2 + 1], s1);
          }
          const double target = (s0 + s1) * dinv[k];
          const double next = target > 0.0 ? target : 0.0;
          const double d_old = h[k] - target, d_new = next - target;
          gain = fma(G[k * R + k], d_old * d_old - d_new * d_new, gain);
          h[k] = next;
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k < r) {
          Hn[(long)k * N + t] = h[k];
          bad |= !isfinite(h[k]);
        }
    }
    const double total = block_sum(gain, red);
    if (sweep == 1) first = total;
    if (sweep >= max_sweeps || total <= stall * (first < 0.0 ? 0.0 : first)) break;
    __syncthreads();   // Hn of this sweep visible to the next
  }
  if (__syncthreads_or(bad)) *nf = 1;
  return sweep;
}

// E-ANLS inner solve (active_set_solve, nnls.hpp:259-406) on r × N columns: G (R × R, shared),
// C and the warm start H0 (r × N, global) → Hn.  bpp::solve_fast_col — the per-run engine's
// lane-parallel FP64 solver — on BPP_WARPS warps, one column per warp at a time, its shared
// memory carved out of WS (the staged-factor region, free after the cross product).  Returns
// the solve rounds (max over the columns); *status = NoConvergence past 3·r·N exchanges
// (nnls.hpp:384-387), NonFiniteIterate on a non-finite solution (engine.hpp:334-337).
constexpr int BPP_WARPS = 6;
constexpr int BPP_LDL = 33;
__host__ __device__ constexpr int bpp_ws_doubles() {
  return 32 * BPP_LDL + BPP_WARPS * (32 * BPP_LDL + 64) + (BPP_WARPS * 32 + 528 + 1) / 2;
}
static_assert(bpp_ws_doubles() <= SMEM_FACTOR, "BPP workspace must fit the staged-factor region");

template <int R>
ENMF_DEV int bpp_solve(const double* G, const double* C, const double* H0, double* Hn, int r, int N, double* WS,
                       double* red, int* status) {
  __shared__ unsigned long long sh_exch;
  __shared__ int sh_rounds, sh_nf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();                                   // WS (the staged factor) no longer read
  const int gld = r | 1;
  double* Gs = WS;
  int* fidx0 = reinterpret_cast<int*>(WS + 32 * BPP_LDL + BPP_WARPS * (32 * BPP_LDL + 64));
  int* tri = fidx0 + BPP_WARPS * 32;
  for (int e = threadIdx.x; e < r * r; e += NT) Gs[(e / r) * gld + e % r] = G[(e / r) * R + e % r];
  bpp::fill_tri(tri, NW);
  double mx = 0.0;                                   // max |C| (feas_tol, nnls.hpp:271)
  for (long e = threadIdx.x; e < (long)r * N; e += NT) {
    const double v = fabs(C[e]);
    mx = mx < v ? v : mx;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) red[warp] = mx;
  if (threadIdx.x == 0) {
    sh_exch = 0;
    sh_rounds = 0;
    sh_nf = 0;
  }
  __syncthreads();
  double cmax = red[0];
  for (int i = 1; i < NW; ++i) cmax = fmax(cmax, red[i]);
  double maxd = 0.0;
  for (int i = 0; i < r; ++i) maxd = (maxd < Gs[i * gld + i]) ? Gs[i * gld + i] : maxd;
  __syncthreads();
  if (warp < BPP_WARPS) {
    bpp::FastCol w;
    w.Gs = Gs;
    w.gld = gld;
    w.tri = tri;
    w.L = WS + 32 * BPP_LDL + warp * (32 * BPP_LDL + 64);
    w.xs = w.L + 32 * BPP_LDL;
    w.invd = w.xs + 32;
    w.fidx = fidx0 + warp * 32;
    w.r = r;
    w.pivot_floor = 1e-12 * maxd;
    w.feas_tol = 1e-12 * (1.0 + cmax);
    w.limit = 3ULL * (unsigned long long)r * (unsigned long long)N;
    unsigned long long ex = 0;
    int rounds = 0, nf = 0;
    for (int col = warp; col < N; col += BPP_WARPS) {
      unsigned long long e;
      int f;
      const int sv = bpp::solve_fast_col(w, C, H0, Hn, N, col, &e, &f);
      ex += e;
      rounds = max(rounds, sv);
      nf |= f;
    }
    if (lane == 0) {
      atomicAdd(&sh_exch, ex);
      atomicMax(&sh_rounds, rounds);
      atomicOr(&sh_nf, nf);
    }
  }
  __syncthreads();
  const unsigned long long ex = sh_exch;
  const int rounds = sh_rounds, nf = sh_nf;
  __syncthreads();
  if (ex > 3ULL * (unsigned long long)r * (unsigned long long)N) *status = ENMF_NO_CONVERGENCE;
  else if (nf) *status = ENMF_NON_FINITE;
  return rounds;
}

// out = next + beta (next − prev) [+ clamp]
ENMF_DEV void extrap(const double* next, const double* prev, double beta, long count, bool clamp, double* out) {
  for (long i = threadIdx.x; i < count; i += NT) {
    const double nv = next[i];
    double v = fma(beta, nv - prev[i], nv);
    if (clamp) v = v > 0.0 ? v : 0.0;
    out[i] = v;
  }
}
ENMF_DEV void copy(const double* src, long count, double* dst) {
  for (long i = threadIdx.x; i < count; i += NT) dst[i] = src[i];
}

// fast_error (engine.hpp:121-136): sqrt(max(0, ||X||² − 2⟨Wᵀ, P⟩ + ⟨GW, GT⟩)), double-double;
// GW, GT are R × R (zero padding).
template <int R>
ENMF_DEV double fast_error(double nxx_hi, double nxx_lo, const double* WT, const double* P, long rm,
                           const double* GW, const double* GT, double* red) {
  double hi = 0.0, lo = 0.0;
  for (long i = threadIdx.x; i < rm; i += NT) {
    const double p = -2.0 * WT[i] * P[i];
    const double e = fma(-2.0 * WT[i], P[i], -p);
    double s, t;
    dd_two_sum(hi, p, s, t);
    hi = s;
    lo += t + e;
  }
  for (int i = threadIdx.x; i < R * R; i += NT) {
    const double p = GW[i] * GT[i];
    const double e = fma(GW[i], GT[i], -p);
    double s, t;
    dd_two_sum(hi, p, s, t);
    hi = s;
    lo += t + e;
  }
  block_dd_sum(hi, lo, red);
  double s, t;
  dd_two_sum(nxx_hi, hi, s, t);
  const double v = s + (t + nxx_lo + lo);
  return sqrt(v > 0.0 ? v : 0.0);
}

template <int R>
__global__ void __launch_bounds__(NT, 2) run(Args a) {
  extern __shared__ __align__(16) double sm[];
  double* SF = sm;                             // staged factor (max(m, n) × R)
  double* GA = SF + SMEM_FACTOR;               // R × R Grams
  double* GB = GA + R * R;
  double* GC = GB + R * R;
  double* GZ = GC + R * R;                     // Gauss-Seidel copy of the Gram in use
  double* DI = GZ + R * R;                     // 1 / G_kk
  __shared__ double red[2 * NW + 2];
  __shared__ int sh_bad[RMAX];
  __shared__ int sh_nb;
  const int m = a.m, n = a.n, r = a.r;
  const long rm = (long)r * m, rn = (long)r * n;
  double* ws = a.ws + (long)blockIdx.x * ws_doubles(m, n, r);
  double* WT = ws;
  double* WyT = WT + rm;
  double* WnT = WyT + rm;
  double* P = WnT + rm;
  double* H = P + rm;
  double* Hy = H + rn;
  double* Hn = Hy + rn;
  double* CH = Hn + rn;
  const enmf_gpu_config& cfg = a.cfg;
  const bool ext = cfg.extrapolation_enabled != 0;
  const bool lit = cfg.hp == 1 && cfg.literal_hp1_order && ext;

  for (long run = blockIdx.x; run < a.count; run += gridDim.x) {
    const double* X = a.x + run * (long)m * n;
    enmf_gpu_iter* recs = a.recs + run * (long)a.cap;
    // ---- prologue (engine.hpp:461-503): factors, ||X||², e(0)
    for (long e = threadIdx.x; e < rm; e += NT) {        // Wᵀ (r × m) from W0 (m × r)
      const int k = (int)(e / m), i = (int)(e % m);
      const double v = a.w0[run * rm + (long)i * r + k];
      WT[e] = v;
      WyT[e] = v;
    }
    for (long e = threadIdx.x; e < rn; e += NT) {
      const double v = a.h0[run * rn + e];
      H[e] = v;
      Hy[e] = v;
    }
    double nh = 0.0, nl = 0.0;
    for (long e = threadIdx.x; e < (long)m * n; e += NT) {
      const double v = __ldg(X + e);
      const double p = v * v, pe = fma(v, v, -p);
      double s, t;
      dd_two_sum(nh, p, s, t);
      nh = s;
      nl += t + pe;
    }
    block_dd_sum(nh, nl, red);
    const double nx = sqrt(nh + nl);
    __syncthreads();
    stage_t<R>(H, r, n, SF);
    __syncthreads();
    gram_t<R>(SF, n, GB);                                // H0 H0ᵀ
    cross_txt<R>(SF, X, m, n, r, P);                     // H0 Xᵀ
    __syncthreads();                                     // every thread done with the staged H0
    stage_t<R>(WT, r, m, SF);
    __syncthreads();
    gram_t<R>(SF, m, GA);                                // W0ᵀ W0
    double err_prev = fast_error<R>(nh, nl, WT, P, rm, GA, GB, red);
    double beta = cfg.beta0, beta_bar = 1.0, beta_prev = cfg.beta0;
    int status = ENMF_OK;
    if (threadIdx.x == 0 && a.cap > 0) {
      enmf_gpu_iter rec{};
      rec.iteration = 0;
      rec.error = err_prev;
      rec.relative_error = nx > 0.0 ? err_prev / nx : 0.0;
      rec.beta = ext ? cfg.beta0 : 0.0;
      recs[0] = rec;
    }
    int nrec = a.cap > 0 ? 1 : 0;
    for (unsigned long long k = 1; k <= cfg.max_outer_iterations; ++k) {
      const double b = ext ? beta : 0.0;
      enmf_gpu_iter rec{};
      rec.iteration = k;
      rec.beta = b;
      int mod = 0, nf = 0;
      // ---- H update (engine.hpp:323-337)
      __syncthreads();
      stage_t<R>(WyT, r, m, SF);
      __syncthreads();
      if (gram_reinit<R>(WyT, SF, r, m, GA, cfg.reinit_seed, 2 * k, &mod, sh_bad, &sh_nb)) { status = ENMF_NO_CONVERGENCE; break; }
      if (threadIdx.x == 0 && mod) rec.reinit_events |= 1;
      cross_wx<R>(SF, X, m, n, r, CH);
      if (cfg.inner_h == ENMF_INNER_EXACT) {
        int st = ENMF_OK;
        __syncthreads();                                 // CH complete
        rec.inner_h_count = bpp_solve<R>(GA, CH, Hy, Hn, r, n, SF, red, &st);
        if (st != ENMF_OK) { status = st; break; }
      } else {
        hals_prep<R>(GA, r, GZ, DI);                     // (ends with a block barrier: CH complete)
        rec.inner_h_count = hals<R>(GA, GZ, DI, CH, Hy, Hn, r, n, a.ms_h, cfg.inner_stall_fraction, red, &nf);
        if (__syncthreads_or(nf)) { status = ENMF_NON_FINITE; break; }
      }
      __syncthreads();
      // ---- early H extrapolation (:340-347)
      if (cfg.hp >= 2) {
        if (ext) extrap(Hn, H, b, rn, cfg.hp == 3, Hy);
        else copy(Hn, rn, Hy);
      }
      __syncthreads();
      // ---- W update (:353-379): T = H_y (hp ≥ 2, or literal hp1 with extrapolation) else H_n
      double* T = (cfg.hp >= 2 || lit) ? Hy : Hn;
      stage_t<R>(T, r, n, SF);
      __syncthreads();
      mod = 0;
      if (gram_reinit<R>(T, SF, r, n, GB, cfg.reinit_seed, 2 * k + 1, &mod, sh_bad, &sh_nb)) { status = ENMF_NO_CONVERGENCE; break; }
      if (threadIdx.x == 0 && mod) rec.reinit_events |= 2;
      cross_txt<R>(SF, X, m, n, r, P);
      if (cfg.inner_w == ENMF_INNER_EXACT) {
        int st = ENMF_OK;
        __syncthreads();                                 // P complete
        rec.inner_w_count = bpp_solve<R>(GB, P, WyT, WnT, r, m, SF, red, &st);
        if (st != ENMF_OK) { status = st; break; }
      } else {
        hals_prep<R>(GB, r, GZ, DI);
        nf = 0;
        rec.inner_w_count = hals<R>(GB, GZ, DI, P, WyT, WnT, r, m, a.ms_w, cfg.inner_stall_fraction, red, &nf);
        if (__syncthreads_or(nf)) { status = ENMF_NON_FINITE; break; }
      }
      __syncthreads();
      // ---- W extrapolation, late H extrapolation (:386-397)
      if (ext) extrap(WnT, WT, b, rm, false, WyT);
      else copy(WnT, rm, WyT);
      if (cfg.hp == 1) {
        if (ext) extrap(Hn, H, b, rn, false, Hy);
        else copy(Hn, rn, Hy);
      }
      __syncthreads();
      // ---- error (:402-416)
      stage_t<R>(WnT, r, m, SF);
      __syncthreads();
      gram_t<R>(SF, m, GC);                              // W_nᵀ W_n
      double err;
      if (lit) {                                         // fresh H_y products (:403-409)
        stage_t<R>(Hy, r, n, SF);
        __syncthreads();
        gram_t<R>(SF, n, GA);
        cross_txt<R>(SF, X, m, n, r, P);                 // H_y Xᵀ (P is free after the W update)
        __syncthreads();
        err = fast_error<R>(nh, nl, WnT, P, rm, GC, GA, red);
      } else {
        err = fast_error<R>(nh, nl, WnT, P, rm, GC, GB, red);
      }
      if (!isfinite(err)) { status = ENMF_NON_FINITE; break; }
      // ---- restart / accept, update_beta (:420-439, 88-99)
      const bool restart = err > err_prev;
      if (restart) {
        copy(WT, rm, WyT);
        copy(H, rn, Hy);
      } else {
        copy(WnT, rm, WT);
        copy(Hn, rn, H);
      }
      if (ext) {
        const bool dec = err <= err_prev;
        const double used = beta;
        if (dec) {
          const double gb = cfg.gamma * beta;
          beta = gb < beta_bar ? gb : beta_bar;
          const double gbb = cfg.gamma_bar * beta_bar;
          beta_bar = gbb < 1.0 ? gbb : 1.0;
        } else {
          beta = beta / cfg.eta;
          beta_bar = beta_prev;
        }
        beta_prev = used;
      }
      err_prev = err;
      if (threadIdx.x == 0 && nrec < a.cap) {
        rec.error = err;
        rec.relative_error = nx > 0.0 ? err / nx : 0.0;
        rec.restarted = restart ? 1 : 0;
        recs[nrec] = rec;
      }
      ++nrec;
    }
    __syncthreads();
    // ---- outputs: W (m × r) from Wᵀ, H
    for (long e = threadIdx.x; e < rm; e += NT) {
      const int k = (int)(e / m), i = (int)(e % m);
      a.w_out[run * rm + (long)i * r + k] = WT[e];
    }
    for (long e = threadIdx.x; e < rn; e += NT) a.h_out[run * rn + e] = H[e];
    if (threadIdx.x == 0) {
      a.n_recs[run] = nrec;
      a.status[run] = status;
      a.norm_x[run] = nx;
    }
    __syncthreads();
  }
}

__host__ inline int smem_bytes() { return (SMEM_FACTOR + 4 * RMAX * RMAX + RMAX) * 8; }

// the compile-time rank bound a run uses: r rounded up to a multiple of 8
__host__ inline int rank_class(int r) { return (r + 7) / 8 * 8; }

}  // namespace batch

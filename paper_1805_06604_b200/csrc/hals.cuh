// hals.cuh — multi-sweep A-HALS inner solver (nnls.hpp:111-176) on sm_100a.
//
// One launch = one Gauss-Seidel sweep over all r rows for every right-hand
// side (column).  Columns are independent within a sweep; the
// only coupling is the global stall rule
//     stop if sweep >= max_sweeps  or  gain <= stall_fraction * max(first_gain, 0)
// (nnls.hpp:172-173), evaluated by the last block to finish (fixed-order sum
// of per-block gains -> deterministic) which also drives the CUDA-graph
// conditional WHILE node that repeats the sweep kernel.
//
// Fast kernel: TPC threads per column, each holding S rows of that column in
// registers (row j lives in thread j % TPC, slot j / TPC); the r×r Gram sits
// in shared memory with its diagonal zeroed and permuted so each thread
// streams its own slots with 16-byte broadcast loads.  Per row k:
//     dot = sum_{j != k} G[k][j] h[j]     (4 FMA chains, then xor-shuffle over TPC)
//     target = (C[k][t] - dot) / G[k][k];  h[k] = max(target, 0)
//     gain += G[k][k] * ((h_old - target)^2 - (h_new - target)^2)
// Exact kernel (precision = FP64_EXACT, and the generic path for r > 128):
// one thread per column in the reference's order (j ascending, gkj == 0
// skipped, no FMA) and a second kernel that sums the per-row gains over the
// columns in the reference's sequential order, so the sweep count and the
// iterates are bitwise those of hals_solve.
#pragma once

#include "common.cuh"

namespace hals {

constexpr int NT = 256;

struct Args {
  const double* G;        // r×r
  const double* C;        // r×N, row stride ld
  const double* Hin;      // warm start (read by sweep 1 only)
  double* H;              // r×N output / in-place iterate
  long ld;
  int r, N;
  int max_sweeps;
  double stall;
  HalsCtl* ctl;
  double* part;           // per-block gain partials
  int* part_nf;           // per-block non-finite flags
  double* terms;          // exact kernel: r×N per-row gain terms
  DevState* st;           // nullable
  int side;               // 0: H update, 1: W update (error message / flags)
  unsigned long long cond;  // cudaGraphConditionalHandle (0 = none)
  int use_cond;
};

ENMF_DEV void set_cond(const Args& a, unsigned v) {
  if (a.use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)a.cond, v);
}

// Stall rule + bookkeeping after a sweep whose total gain is `gain`.
ENMF_DEV void finish_sweep(const Args& a, double gain, int nonfinite) {
  HalsCtl* c = a.ctl;
  const int s = c->sweeps + 1;
  c->sweeps = s;
  if (s == 1) c->first_gain = gain;
  c->last_gain = gain;
  const double fg = c->first_gain;
  const bool stop = (s >= a.max_sweeps) || (gain <= __dmul_rn(a.stall, fg < 0.0 ? 0.0 : fg));
  c->cont = stop ? 0 : 1;
  c->nonfinite = nonfinite;
  if (stop && nonfinite && a.st) {
    // NaN guard on the finished iterate (engine.hpp:334-337 / 380-383)
    if (a.st->active) {
      a.st->error_code = ENMF_NON_FINITE;
      a.st->active = 0;
    }
  }
  __threadfence();
  set_cond(a, stop ? 0u : 1u);
}

// Returns true (uniformly) if this launch must do no work.
ENMF_DEV bool sweep_skipped(const Args& a) {
  const bool skip = (a.st && !dev_active(a.st)) || !*(volatile int*)&a.ctl->cont;
  if (skip && blockIdx.x == 0 && threadIdx.x == 0) set_cond(a, 0u);
  return skip;
}

// Last-arriving block: fixed-order sum of the per-block partials.
template <int NTH>
ENMF_DEV void last_block_reduce_n(const Args& a, double block_gain, int block_nf, double* red) {
  __shared__ unsigned s_last;
  if (threadIdx.x == 0) {
    a.part[blockIdx.x] = block_gain;
    a.part_nf[blockIdx.x] = block_nf;
    __threadfence();
    const unsigned prev = atomicAdd(&a.ctl->arrive, 1u);
    s_last = (prev == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double v = 0.0;
  int nf = 0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += NTH) {
    v = __dadd_rn(v, __ldcg(a.part + b));
    nf |= __ldcg(a.part_nf + b);
  }
  const double total = block_reduce_sum_any(v, red);
  nf = __syncthreads_or(nf);
  if (threadIdx.x == 0) {
    a.ctl->arrive = 0;
    finish_sweep(a, total, nf);
  }
}

template <int S, int TPC>
constexpr int smem_bytes() {
  return (S * TPC) * TPC * (S + 2) * 8 + (S * TPC) * 8;
}

template <int S, int TPC>
__global__ void __launch_bounds__(NT) sweep_fast(Args a) {
  constexpr int RMAX = S * TPC;
  constexpr int GROW = TPC * (S + 2);
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;                 // [RMAX][TPC][S+2], diagonal zeroed
  double* Gd = sm + RMAX * GROW;   // diag
  __shared__ double red[NT];

  const int r = a.r;
  for (int e = threadIdx.x; e < RMAX * TPC * S; e += NT) {
    const int k = e / (TPC * S), rem = e % (TPC * S), q = rem / S, s = rem % S;
    const int j = s * TPC + q;
    double v = 0.0;
    if (k < r && j < r && j != k) v = a.G[k * r + j];
    Gs[k * GROW + q * (S + 2) + s] = v;
  }
  for (int k = threadIdx.x; k < RMAX; k += NT) Gd[k] = k < r ? a.G[k * r + k] : 1.0;
  __syncthreads();

  const int q = threadIdx.x % TPC;
  const int t = blockIdx.x * (NT / TPC) + threadIdx.x / TPC;
  const bool valid = t < a.N;
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;

  double h[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int j = s * TPC + q;
    h[s] = (valid && j < r) ? src[(long)j * a.ld + t] : 0.0;
  }
  double gain = 0.0;
  double cnext = (valid) ? a.C[t] : 0.0;
  // Rows k >= r are padding: zero Gram row, unit diagonal, zero cross term,
  // so their update is a no-op (target 0, h stays 0, gain 0); no data-dependent
  // exit keeps the loop fully unrolled and every h[] index static.
#pragma unroll
  for (int k = 0; k < RMAX; ++k) {
    const double ck = cnext;
    if (k + 1 < r && valid) cnext = a.C[(long)(k + 1) * a.ld + t];
    else cnext = 0.0;
    const double2* gk = reinterpret_cast<const double2*>(Gs + k * GROW + q * (S + 2));
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int s2 = 0; s2 < S / 2; ++s2) {
      const double2 gv = gk[s2];
      acc[(2 * s2) & 3] = fma(gv.x, h[2 * s2], acc[(2 * s2) & 3]);
      acc[(2 * s2 + 1) & 3] = fma(gv.y, h[2 * s2 + 1], acc[(2 * s2 + 1) & 3]);
    }
    double dot = __dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3]));
#pragma unroll
    for (int off = 1; off < TPC; off <<= 1) dot = __dadd_rn(dot, __shfl_xor_sync(0xffffffffu, dot, off));
    const double gkk = Gd[k];
    const double target = __ddiv_rn(__dsub_rn(ck, dot), gkk);
    const double next = target > 0.0 ? target : 0.0;
    if (q == (k % TPC)) {
      const double d_old = __dsub_rn(h[k / TPC], target);
      const double d_new = __dsub_rn(next, target);
      gain = fma(gkk, __dsub_rn(__dmul_rn(d_old, d_old), __dmul_rn(d_new, d_new)), gain);
      h[k / TPC] = next;
    }
  }
  int nf = 0;
  if (valid) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int j = s * TPC + q;
      if (j < r) {
        a.H[(long)j * a.ld + t] = h[s];
        nf |= !isfinite(h[s]);
      }
    }
  }
  const double bg = block_reduce_sum<NT>(valid ? gain : 0.0, red);
  nf = __syncthreads_or(nf);
  last_block_reduce_n<NT>(a, bg, nf, red);
}

// ---- tensor-core sweep: blocked Gauss-Seidel on DMMA ----------------------
//
// The r rows are processed in blocks of 8.  For block K = [k0, k0+8) and the 8
// columns a warp owns,
//     S = G[K, :] · H            (DMMA m8n8k4 over j, 4 independent accumulators)
// uses the current H (rows < k0 already updated this sweep, rows >= k0 old), so
//     b_k = C_k - sum_{j != k} G_kj h_j = C_k - S_k + G_kk h_old_k - sum_{i in K, i < k} G_ki (h_new_i - h_old_i)
// and the 8 rows of the block are then finished sequentially with one shuffle
// per row to forward the change δ_i.  H lives in registers in the DMMA
// B-fragment layout: lane (g, t) holds H[4s + t][col g] in slot s.  Per sweep
// this is r·r·N FMAs on the tensor pipe (the reference's r² per column).
constexpr int kDmmaWarps = 14;

template <int RMAX>
constexpr int dmma_smem_bytes() {
  return RMAX * (RMAX + 4) * 8 + 2 * RMAX * 8;
}

template <int RMAX>
__global__ void __launch_bounds__(kDmmaWarps * 32, 1) sweep_dmma(Args a) {
  constexpr int LDG = RMAX + 4;    // conflict-free A-fragment rows
  constexpr int SL = RMAX / 4;     // H slots per lane
  constexpr int NB = RMAX / 8;     // row blocks
  constexpr int NTH = kDmmaWarps * 32;
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;                 // [RMAX][LDG]
  double* Gd = sm + RMAX * LDG;    // G_kk (1 for padding rows)
  double* Gi = Gd + RMAX;          // 1 / G_kk
  __shared__ double red[NTH];

  const int r = a.r;
  for (int e = threadIdx.x; e < RMAX * RMAX; e += NTH) {
    const int k = e / RMAX, j = e % RMAX;
    Gs[k * LDG + j] = (k < r && j < r) ? a.G[k * r + j] : 0.0;
  }
  for (int k = threadIdx.x; k < RMAX; k += NTH) {
    const double d = k < r ? a.G[k * r + k] : 1.0;
    Gd[k] = d;
    Gi[k] = __ddiv_rn(1.0, d);
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long c0 = ((long)blockIdx.x * kDmmaWarps + warp) * 8;
  const long colH = c0 + g;                 // column this lane holds in the H layout
  const bool validH = colH < a.N;
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  double hreg[SL];
#pragma unroll
  for (int s = 0; s < SL; ++s) {
    const int j = 4 * s + t;
    hreg[s] = (validH && j < r) ? src[(long)j * a.ld + colH] : 0.0;
  }
  // S-layout columns of this lane: c0 + 2t + e
  const long colS = c0 + 2 * t;
  const bool v0 = colS < a.N, v1 = colS + 1 < a.N;
  auto loadC = [&](int k, double& x0, double& x1) {
    x0 = (k < r && v0) ? a.C[(long)k * a.ld + colS] : 0.0;
    x1 = (k < r && v1) ? a.C[(long)k * a.ld + colS + 1] : 0.0;
  };
  double cn0, cn1;
  loadC(g, cn0, cn1);
  double gain = 0.0;

#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int k0 = 8 * b;
    const double cc0 = cn0, cc1 = cn1;
    if (b + 1 < NB) loadC(k0 + 8 + g, cn0, cn1);
    // S = G[K, :] · H
    double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    const double* ga = Gs + (k0 + g) * LDG + t;
#pragma unroll
    for (int s = 0; s < SL; ++s) dmma884(acc[s & 3][0], acc[s & 3][1], ga[4 * s], hreg[s]);
    const double S0 = __dadd_rn(__dadd_rn(acc[0][0], acc[1][0]), __dadd_rn(acc[2][0], acc[3][0]));
    const double S1 = __dadd_rn(__dadd_rn(acc[0][1], acc[1][1]), __dadd_rn(acc[2][1], acc[3][1]));
    // h_old of (row k0+g, cols colS, colS+1) from the H layout
    const int srcA0 = (2 * t) * 4 + (g & 3), srcA1 = (2 * t + 1) * 4 + (g & 3);
    const double lo0 = __shfl_sync(0xffffffffu, hreg[2 * b], srcA0);
    const double lo1 = __shfl_sync(0xffffffffu, hreg[2 * b], srcA1);
    const double hi0 = __shfl_sync(0xffffffffu, hreg[2 * b + 1], srcA0);
    const double hi1 = __shfl_sync(0xffffffffu, hreg[2 * b + 1], srcA1);
    const double ho0 = g < 4 ? lo0 : hi0, ho1 = g < 4 ? lo1 : hi1;
    const int k = k0 + g;
    const double gkk = Gd[k], ginv = Gi[k];
    const double b0 = fma(gkk, ho0, __dsub_rn(cc0, S0));
    const double b1 = fma(gkk, ho1, __dsub_rn(cc1, S1));
    double gblk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) gblk[i] = Gs[k * LDG + k0 + i];
    double corr0 = 0.0, corr1 = 0.0, hn0 = ho0, hn1 = ho1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double d0 = 0.0, d1 = 0.0;
      if (g == i) {
        const double t0 = __dmul_rn(__dsub_rn(b0, corr0), ginv);
        const double t1 = __dmul_rn(__dsub_rn(b1, corr1), ginv);
        hn0 = t0 > 0.0 ? t0 : 0.0;
        hn1 = t1 > 0.0 ? t1 : 0.0;
        d0 = __dsub_rn(hn0, ho0);
        d1 = __dsub_rn(hn1, ho1);
        const double o0 = __dsub_rn(ho0, t0), n0 = __dsub_rn(hn0, t0);
        const double o1 = __dsub_rn(ho1, t1), n1 = __dsub_rn(hn1, t1);
        gain = fma(gkk, __dsub_rn(__dmul_rn(o0, o0), __dmul_rn(n0, n0)), gain);
        gain = fma(gkk, __dsub_rn(__dmul_rn(o1, o1), __dmul_rn(n1, n1)), gain);
      }
      if (i < 7) {
        const double e0 = __shfl_sync(0xffffffffu, d0, i * 4 + t);
        const double e1 = __shfl_sync(0xffffffffu, d1, i * 4 + t);
        if (g > i) {
          corr0 = fma(gblk[i], e0, corr0);
          corr1 = fma(gblk[i], e1, corr1);
        }
      }
    }
    // back to the H layout: lane (g', t') takes rows k0+t' and k0+4+t' of column g'
    const int srcB_lo = t * 4 + (g >> 1), srcB_hi = (t + 4) * 4 + (g >> 1);
    const double x0lo = __shfl_sync(0xffffffffu, hn0, srcB_lo);
    const double x1lo = __shfl_sync(0xffffffffu, hn1, srcB_lo);
    const double x0hi = __shfl_sync(0xffffffffu, hn0, srcB_hi);
    const double x1hi = __shfl_sync(0xffffffffu, hn1, srcB_hi);
    hreg[2 * b] = (g & 1) ? x1lo : x0lo;
    hreg[2 * b + 1] = (g & 1) ? x1hi : x0hi;
  }
  int nf = 0;
  if (validH) {
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      const int j = 4 * s + t;
      if (j < r) {
        a.H[(long)j * a.ld + colH] = hreg[s];
        nf |= !isfinite(hreg[s]);
      }
    }
  }
  const double bg = block_reduce_sum_any(gain, red);
  nf = __syncthreads_or(nf);
  last_block_reduce_n<NTH>(a, bg, nf, red);
}

// ---- persistent tensor-core sweep (default) ---------------------------------
//
// Same blocked Gauss-Seidel as sweep_dmma, restructured after profiling
// (profiles/r01_sweep_dmma_v1.txt: spills, i-cache misses from the fully
// unrolled block loop, per-CTA Gram reload, predicated-off FP64 work):
//   * persistent: one CTA per SM walks the column tiles, the Gram is staged into
//     shared memory once per launch with cp.async;
//   * rolled block loop: the current block's rows always sit in slots 0/1 of
//     the register file image of H (rotated by two slots after each block), the
//     A-fragment column is indexed by the rotation instead;
//   * the gain is evaluated after the sequential 8-row pass, by all lanes.
template <int RMAX>
__global__ void __launch_bounds__(kDmmaWarps * 32, 1) sweep_dmma_p(Args a, int ntiles) {
  constexpr int LDG = RMAX + 4;
  constexpr int SL = RMAX / 4;
  constexpr int NB = RMAX / 8;
  constexpr int NTH = kDmmaWarps * 32;
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;
  double* Gd = sm + RMAX * LDG;
  double* Gi = Gd + RMAX;
  __shared__ double red[NTH];

  const int r = a.r;
  {
    // cp.async the r×r Gram into padded rows; padding zero-filled
    constexpr int CH = RMAX / 2;  // 16-byte chunks per padded row
    const bool vec = (r % 2 == 0) && (((uintptr_t)a.G & 15) == 0);
    for (int e = threadIdx.x; e < RMAX * CH; e += NTH) {
      const int k = e / CH, j = (e % CH) * 2;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(Gs + k * LDG + j);
      if (vec) {
        const int valid = (k < r && j < r) ? 16 : 0;
        const double* srcp = valid ? a.G + (long)k * r + j : a.G;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(srcp), "r"(valid));
      } else {
        Gs[k * LDG + j] = (k < r && j < r) ? a.G[(long)k * r + j] : 0.0;
        Gs[k * LDG + j + 1] = (k < r && j + 1 < r) ? a.G[(long)k * r + j + 1] : 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    for (int k = threadIdx.x; k < RMAX; k += NTH) {
      const double d = k < r ? a.G[(long)k * r + k] : 1.0;
      Gd[k] = d;
      Gi[k] = __ddiv_rn(1.0, d);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  double gain = 0.0;
  int nf = 0;
  bool first = true;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c0 = ((long)tile * kDmmaWarps + warp) * 8;
    const long colH = c0 + g;
    const bool validH = colH < a.N;
    double hreg[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      const int j = 4 * s + t;
      hreg[s] = (validH && j < r) ? src[(long)j * a.ld + colH] : 0.0;
    }
    const long colS = c0 + 2 * t;
    const bool v0 = colS < a.N, v1 = colS + 1 < a.N;
    double cn0 = (g < r && v0) ? a.C[(long)g * a.ld + colS] : 0.0;
    double cn1 = (g < r && v1) ? a.C[(long)g * a.ld + colS + 1] : 0.0;
    if (first) {
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
      first = false;
    }
    const int srcA0 = (2 * t) * 4 + (g & 3), srcA1 = (2 * t + 1) * 4 + (g & 3);
    const int srcB_lo = t * 4 + (g >> 1), srcB_hi = (t + 4) * 4 + (g >> 1);
#pragma unroll 1
    for (int b = 0; b < NB; ++b) {
      const int k0 = 8 * b;
      const int k = k0 + g;
      const double cc0 = cn0, cc1 = cn1;
      if (b + 1 < NB) {
        const int kn = k + 8;
        cn0 = (kn < r && v0) ? a.C[(long)kn * a.ld + colS] : 0.0;
        cn1 = (kn < r && v1) ? a.C[(long)kn * a.ld + colS + 1] : 0.0;
      }
      // S = G[K, :] · H ; slot s holds rows 4·((s + 2b) mod SL) + t
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      const double* ga = Gs + k * LDG + t;
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const int js = (s + 2 * b) & (SL - 1);
        dmma884(acc[s & 3][0], acc[s & 3][1], ga[4 * js], hreg[s]);
      }
      const double S0 = __dadd_rn(__dadd_rn(acc[0][0], acc[1][0]), __dadd_rn(acc[2][0], acc[3][0]));
      const double S1 = __dadd_rn(__dadd_rn(acc[0][1], acc[1][1]), __dadd_rn(acc[2][1], acc[3][1]));
      const double lo0 = __shfl_sync(0xffffffffu, hreg[0], srcA0);
      const double lo1 = __shfl_sync(0xffffffffu, hreg[0], srcA1);
      const double hi0 = __shfl_sync(0xffffffffu, hreg[1], srcA0);
      const double hi1 = __shfl_sync(0xffffffffu, hreg[1], srcA1);
      const double ho0 = g < 4 ? lo0 : hi0, ho1 = g < 4 ? lo1 : hi1;
      const double gkk = Gd[k], ginv = Gi[k];
      const double b0 = fma(gkk, ho0, __dsub_rn(cc0, S0));
      const double b1 = fma(gkk, ho1, __dsub_rn(cc1, S1));
      double corr0 = 0.0, corr1 = 0.0, hn0 = ho0, hn1 = ho1, t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double gki = Gs[k * LDG + k0 + i];
        double d0 = 0.0, d1 = 0.0;
        if (g == i) {
          t0 = __dmul_rn(__dsub_rn(b0, corr0), ginv);
          t1 = __dmul_rn(__dsub_rn(b1, corr1), ginv);
          hn0 = t0 > 0.0 ? t0 : 0.0;
          hn1 = t1 > 0.0 ? t1 : 0.0;
          d0 = __dsub_rn(hn0, ho0);
          d1 = __dsub_rn(hn1, ho1);
        }
        if (i < 7) {
          const double e0 = __shfl_sync(0xffffffffu, d0, i * 4 + t);
          const double e1 = __shfl_sync(0xffffffffu, d1, i * 4 + t);
          if (g > i) {
            corr0 = fma(gki, e0, corr0);
            corr1 = fma(gki, e1, corr1);
          }
        }
      }
      {
        const double o0 = __dsub_rn(ho0, t0), n0 = __dsub_rn(hn0, t0);
        const double o1 = __dsub_rn(ho1, t1), n1 = __dsub_rn(hn1, t1);
        gain = fma(gkk, __dsub_rn(__dmul_rn(o0, o0), __dmul_rn(n0, n0)), gain);
        gain = fma(gkk, __dsub_rn(__dmul_rn(o1, o1), __dmul_rn(n1, n1)), gain);
      }
      const double x0lo = __shfl_sync(0xffffffffu, hn0, srcB_lo);
      const double x1lo = __shfl_sync(0xffffffffu, hn1, srcB_lo);
      const double x0hi = __shfl_sync(0xffffffffu, hn0, srcB_hi);
      const double x1hi = __shfl_sync(0xffffffffu, hn1, srcB_hi);
      const double new_lo = (g & 1) ? x1lo : x0lo;
      const double new_hi = (g & 1) ? x1hi : x0hi;
      // rotate: the next block's rows move into slots 0/1, this block's go last
#pragma unroll
      for (int s = 0; s + 2 < SL; ++s) hreg[s] = hreg[s + 2];
      hreg[SL - 2] = new_lo;
      hreg[SL - 1] = new_hi;
    }
    // after NB blocks the rotation is back to the identity (2·NB = SL)
    if (validH) {
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const int j = 4 * s + t;
        if (j < r) {
          a.H[(long)j * a.ld + colH] = hreg[s];
          nf |= !isfinite(hreg[s]);
        }
      }
    }
  }
  if (first) {
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
  }
  const double bg = block_reduce_sum_any(gain, red);
  nf = __syncthreads_or(nf);
  last_block_reduce_n<NTH>(a, bg, nf, red);
}

// ---- bitwise-faithful sweep (hals_row_update_impl order) -----------------
__global__ void __launch_bounds__(NT) sweep_exact(Args a) {
  if (sweep_skipped(a)) return;
  const int t = blockIdx.x * NT + threadIdx.x;
  if (t >= a.N) return;
  const int r = a.r;
  if (a.ctl->sweeps == 0) {
    for (int j = 0; j < r; ++j) a.H[(long)j * a.ld + t] = a.Hin[(long)j * a.ld + t];
  }
  for (int k = 0; k < r; ++k) {
    const double gkk = a.G[k * r + k];
    double b = a.C[(long)k * a.ld + t];
    for (int j = 0; j < r; ++j) {
      if (j == k) continue;
      const double gkj = a.G[k * r + j];
      if (gkj == 0.0) continue;
      b = __dsub_rn(b, __dmul_rn(gkj, a.H[(long)j * a.ld + t]));
    }
    const double hk = a.H[(long)k * a.ld + t];
    const double target = __ddiv_rn(b, gkk);
    const double next = target > 0.0 ? target : 0.0;
    const double d_old = __dsub_rn(hk, target);
    const double d_new = __dsub_rn(next, target);
    a.terms[(long)k * a.N + t] = __dsub_rn(__dmul_rn(d_old, d_old), __dmul_rn(d_new, d_new));
    a.H[(long)k * a.ld + t] = next;
  }
}

// gain = sum_k G[k][k] * (sum_t terms[k][t])  in the reference's order.
__global__ void __launch_bounds__(NT) gain_exact(Args a) {
  if ((a.st && !dev_active(a.st)) || !*(volatile int*)&a.ctl->cont) return;  // sweep_exact set cond
  __shared__ double rowgain[1024];
  const int r = a.r;
  for (int k = threadIdx.x; k < r; k += NT) {
    double gk = 0.0;
    const double* tk = a.terms + (long)k * a.N;
    for (int t = 0; t < a.N; ++t) gk = __dadd_rn(gk, tk[t]);
    rowgain[k < 1024 ? k : 1023] = __dmul_rn(a.G[k * r + k], gk);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double gain = 0.0;
    for (int k = 0; k < r; ++k) gain = __dadd_rn(gain, rowgain[k]);
    int nf = 0;
    for (int k = 0; k < r && !nf; ++k)
      for (int t = 0; t < a.N; ++t)
        if (!isfinite(a.H[(long)k * a.ld + t])) { nf = 1; break; }
    finish_sweep(a, gain, nf);
  }
}

// Resets the control block at the start of a solve.
__global__ void reset_ctl(HalsCtl* c, const DevState* st) {
  if (st && !dev_active(st)) return;
  c->first_gain = 0.0;
  c->last_gain = 0.0;
  c->sweeps = 0;
  c->cont = 1;
  c->nonfinite = 0;
  c->arrive = 0;
}

}  // namespace hals

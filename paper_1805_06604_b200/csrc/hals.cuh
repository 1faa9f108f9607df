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
#include "dist.cuh"

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
  const dist::View* dv;     // multi-GPU: all-reduce the sweep gain across ranks (nullable)
  const double* Gf;         // sweep_ws: Gram in A-fragment order (ws_prep)
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
  double total = block_reduce_sum_any(v, red);
  nf = __syncthreads_or(nf);
  if (threadIdx.x == 0) {
    a.ctl->arrive = 0;
    if (a.dv) dist::allreduce_gain(*a.dv, total, nf, &total, &nf);  // global stall rule
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
  __shared__ double red[NTH + 33];

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
template <int RMAX, int UB = 1, int NW = kDmmaWarps>
__global__ void __launch_bounds__(NW * 32, 1) sweep_dmma_p(Args a, int ntiles) {
  constexpr int LDG = RMAX + 4;
  constexpr int SL = RMAX / 4;
  constexpr int NB = RMAX / 8;
  constexpr int NTH = NW * 32;
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;
  double* Gd = sm + RMAX * LDG;
  double* Gi = Gd + RMAX;
  __shared__ double red[NTH + 33];

  const int r = a.r;
  {
    // cp.async the r×r Gram into padded rows, each row block's columns rotated
    // by its own offset:  Gs[k][c] = G[k][(c + 8·(k/8)) mod RMAX]  (padding zero).
    // With H's register image rotated by 8 slots per 4 blocks, every A-fragment
    // and in-block coupling address below is a compile-time offset.
    constexpr int CH = RMAX / 2;  // 16-byte chunks per padded row
    const bool vec = (r % 2 == 0) && (((uintptr_t)a.G & 15) == 0);
    for (int e = threadIdx.x; e < RMAX * CH; e += NTH) {
      const int k = e / CH, c = (e % CH) * 2;
      const int j = (c + 8 * (k / 8)) & (RMAX - 1);
      const unsigned dst = (unsigned)__cvta_generic_to_shared(Gs + k * LDG + c);
      if (vec) {
        const int valid = (k < r && j < r) ? 16 : 0;
        const double* srcp = valid ? a.G + (long)k * r + j : a.G;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(srcp), "r"(valid));
      } else {
        Gs[k * LDG + c] = (k < r && j < r) ? a.G[(long)k * r + j] : 0.0;
        Gs[k * LDG + c + 1] = (k < r && j + 1 < r) ? a.G[(long)k * r + j + 1] : 0.0;
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
    const long c0 = ((long)tile * NW + warp) * 8;
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
    const double* gbase = Gs + g * LDG + t;
#pragma unroll 1
    for (int q = 0; q < NB / UB; ++q) {
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int b = UB * q + u;
      const int k0 = 8 * b;
      const int k = k0 + g;
      const double cc0 = cn0, cc1 = cn1;
      if (b + 1 < NB) {
        const int kn = k + 8;
        cn0 = (kn < r && v0) ? a.C[(long)kn * a.ld + colS] : 0.0;
        cn1 = (kn < r && v1) ? a.C[(long)kn * a.ld + colS + 1] : 0.0;
      }
      // S = G[K, :] · H ; slot s holds original slot (s + 8q) mod SL, i.e. rows
      // 4((s + 8q) mod SL) + t, stored at rotated column (4s - 8u) mod RMAX + t.
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      const double* ga = gbase + k0 * LDG;
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const int col = (4 * s - 8 * u + RMAX) & (RMAX - 1);
        dmma884(acc[s & 3][0], acc[s & 3][1], ga[col], hreg[s]);
      }
      const double S0 = __dadd_rn(__dadd_rn(acc[0][0], acc[1][0]), __dadd_rn(acc[2][0], acc[3][0]));
      const double S1 = __dadd_rn(__dadd_rn(acc[0][1], acc[1][1]), __dadd_rn(acc[2][1], acc[3][1]));
      const double lo0 = __shfl_sync(0xffffffffu, hreg[2 * u], srcA0);
      const double lo1 = __shfl_sync(0xffffffffu, hreg[2 * u], srcA1);
      const double hi0 = __shfl_sync(0xffffffffu, hreg[2 * u + 1], srcA0);
      const double hi1 = __shfl_sync(0xffffffffu, hreg[2 * u + 1], srcA1);
      const double ho0 = g < 4 ? lo0 : hi0, ho1 = g < 4 ? lo1 : hi1;
      const double gkk = Gd[k], ginv = Gi[k];
      const double b0 = fma(gkk, ho0, __dsub_rn(cc0, S0));
      const double b1 = fma(gkk, ho1, __dsub_rn(cc1, S1));
      double corr0 = 0.0, corr1 = 0.0, hn0 = ho0, hn1 = ho1, t0 = 0.0, t1 = 0.0;
      const double* gk = Gs + k * LDG;  // G[k][k0 + i] sits at rotated column i
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double gki = gk[i];
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
      hreg[2 * u] = (g & 1) ? x1lo : x0lo;
      hreg[2 * u + 1] = (g & 1) ? x1hi : x0hi;
    }
    // rotate the register image by 8 slots: the next 4 blocks' rows move to slots 0..7
    {
      double tmp[2 * UB];
#pragma unroll
      for (int s = 0; s < 2 * UB; ++s) tmp[s] = hreg[s];
#pragma unroll
      for (int s = 0; s + 2 * UB < SL; ++s) hreg[s] = hreg[s + 2 * UB];
#pragma unroll
      for (int s = 0; s < 2 * UB; ++s) hreg[SL - 2 * UB + s] = tmp[s];
    }
    }
    // after NB/4 groups the rotation is back to the identity (8·NB/4 = SL)
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

// ---- transposed-tile tensor-core sweep (default) -----------------------------
//
// As sweep_dmma_p, but the DMMA computes the block's products column-major,
//     D[col][row] = sum_j H[j][col] · G[k0+row][j]      (A = H fragment, B = G fragment),
// so lane (g, t) ends up with rows k0+2t, k0+2t+1 of column g.  In the
// sequential 8-row pass every active lane then finishes ONE (row, column)
// element per step and 8 lanes (one per column) are active instead of 4
// lanes × 2 columns: half the FP64 instructions of the pass.  δ of a row is
// forwarded inside the lane quad of its column.
template <int RMAX, int UB, int NW>
__global__ void __launch_bounds__(NW * 32, 1) sweep_dmma_t(Args a, int ntiles) {
  constexpr int LDG = RMAX + 4;
  constexpr int SL = RMAX / 4;
  constexpr int NB = RMAX / 8;
  constexpr int NTH = NW * 32;
  static_assert(NB % UB == 0, "row blocks per group");
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;
  double* Gd = sm + RMAX * LDG;
  double* Gi = Gd + RMAX;
  __shared__ double red[NTH + 33];

  const int r = a.r;
  {
    // Gs[k][c] = G[k][(c + 8·(k/8)) mod RMAX] (see sweep_dmma_p), zero padding
    constexpr int CH = RMAX / 2;
    const bool vec = (r % 2 == 0) && (((uintptr_t)a.G & 15) == 0);
    for (int e = threadIdx.x; e < RMAX * CH; e += NTH) {
      const int k = e / CH, c = (e % CH) * 2;
      const int j = (c + 8 * (k / 8)) & (RMAX - 1);
      const unsigned dst = (unsigned)__cvta_generic_to_shared(Gs + k * LDG + c);
      if (vec) {
        const int valid = (k < r && j < r) ? 16 : 0;
        const double* srcp = valid ? a.G + (long)k * r + j : a.G;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(srcp), "r"(valid));
      } else {
        Gs[k * LDG + c] = (k < r && j < r) ? a.G[(long)k * r + j] : 0.0;
        Gs[k * LDG + c + 1] = (k < r && j + 1 < r) ? a.G[(long)k * r + j + 1] : 0.0;
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
  // gather sources (H layout -> tile layout): rows k0+2t+e live in lane (g, (2t+e)&3)
  const int sg0 = g * 4 + ((2 * t) & 3), sg1 = g * 4 + ((2 * t + 1) & 3);
  const bool upper = t >= 2;  // rows k0+4.. (second slot of the block)
  // scatter sources (tile layout -> H layout): row k0+t lives in lane (g, t/2) elem t&1,
  // row k0+4+t in lane (g, 2 + t/2) elem t&1
  const int ss_lo = g * 4 + (t >> 1), ss_hi = g * 4 + 2 + (t >> 1);
  const bool odd = t & 1;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long col = ((long)tile * NW + warp) * 8 + g;   // this lane's column (both layouts)
    const bool valid = col < a.N;
    double hreg[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      const int j = 4 * s + t;
      hreg[s] = (valid && j < r) ? src[(long)j * a.ld + col] : 0.0;
    }
    const double* cp = a.C + col;
    double cn0 = (valid && 2 * t < r) ? cp[(long)(2 * t) * a.ld] : 0.0;
    double cn1 = (valid && 2 * t + 1 < r) ? cp[(long)(2 * t + 1) * a.ld] : 0.0;
    if (first) {
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
      first = false;
    }
    const double* gbase = Gs + g * LDG + t;   // B fragment: G[k0 + g][rotated col + t]
#pragma unroll 1
    for (int q = 0; q < NB / UB; ++q) {
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int b = UB * q + u;
        const int k0 = 8 * b;
        const int ka = k0 + 2 * t;          // this lane's two rows: ka, ka+1
        const double cc0 = cn0, cc1 = cn1;
        if (b + 1 < NB) {
          cn0 = (valid && ka + 8 < r) ? cp[(long)(ka + 8) * a.ld] : 0.0;
          cn1 = (valid && ka + 9 < r) ? cp[(long)(ka + 9) * a.ld] : 0.0;
        }
        double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        const double* gb = gbase + k0 * LDG;
#pragma unroll
        for (int s = 0; s < SL; ++s) {
          const int c = (4 * s - 8 * u + RMAX) & (RMAX - 1);
          dmma884(acc[s & 3][0], acc[s & 3][1], hreg[s], gb[c]);
        }
        const double S0 = __dadd_rn(__dadd_rn(acc[0][0], acc[1][0]), __dadd_rn(acc[2][0], acc[3][0]));
        const double S1 = __dadd_rn(__dadd_rn(acc[0][1], acc[1][1]), __dadd_rn(acc[2][1], acc[3][1]));
        // h_old of rows ka, ka+1 (slot 2u for rows k0..k0+3, 2u+1 for k0+4..k0+7)
        const double xa0 = __shfl_sync(0xffffffffu, hreg[2 * u], sg0);
        const double xb0 = __shfl_sync(0xffffffffu, hreg[2 * u + 1], sg0);
        const double xa1 = __shfl_sync(0xffffffffu, hreg[2 * u], sg1);
        const double xb1 = __shfl_sync(0xffffffffu, hreg[2 * u + 1], sg1);
        const double x0 = upper ? xb0 : xa0, x1 = upper ? xb1 : xa1;
        const double* gk0 = Gs + ka * LDG;        // G[ka][k0 + i] at rotated column i
        const double* gk1 = gk0 + LDG;
        const double g00 = Gd[ka], g11 = Gd[ka + 1];
        const double i00 = Gi[ka], i11 = Gi[ka + 1];
        double b0 = fma(g00, x0, __dsub_rn(cc0, S0));
        double b1 = fma(g11, x1, __dsub_rn(cc1, S1));
        double h0 = x0, h1 = x1, t0 = 0.0, t1 = 0.0;
        // sequential pass: row k0+i is element i&1 of lane t = i/2
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          double d0 = 0.0, d1 = 0.0;
          if (2 * t == i) {
            t0 = __dmul_rn(b0, i00);
            h0 = t0 > 0.0 ? t0 : 0.0;
            d0 = __dsub_rn(h0, x0);
            b1 = fma(-gk1[i], d0, b1);            // row ka+1 sees row ka at once
            t1 = __dmul_rn(b1, i11);
            h1 = t1 > 0.0 ? t1 : 0.0;
            d1 = __dsub_rn(h1, x1);
          }
          if (i < 6) {
            const double e0 = __shfl_sync(0xffffffffu, d0, g * 4 + i / 2);
            const double e1 = __shfl_sync(0xffffffffu, d1, g * 4 + i / 2);
            if (2 * t > i) {
              b0 = fma(-gk0[i], e0, b0);
              b0 = fma(-gk0[i + 1], e1, b0);
              b1 = fma(-gk1[i], e0, b1);
              b1 = fma(-gk1[i + 1], e1, b1);
            }
          }
        }
        {
          const double o0 = __dsub_rn(x0, t0), n0 = __dsub_rn(h0, t0);
          const double o1 = __dsub_rn(x1, t1), n1 = __dsub_rn(h1, t1);
          gain = fma(g00, __dsub_rn(__dmul_rn(o0, o0), __dmul_rn(n0, n0)), gain);
          gain = fma(g11, __dsub_rn(__dmul_rn(o1, o1), __dmul_rn(n1, n1)), gain);
        }
        // back to the H layout
        const double y0 = __shfl_sync(0xffffffffu, h0, ss_lo);
        const double y1 = __shfl_sync(0xffffffffu, h1, ss_lo);
        const double z0 = __shfl_sync(0xffffffffu, h0, ss_hi);
        const double z1 = __shfl_sync(0xffffffffu, h1, ss_hi);
        hreg[2 * u] = odd ? y1 : y0;
        hreg[2 * u + 1] = odd ? z1 : z0;
      }
      if (NB / UB > 1) {
        double tmp[2 * UB];
#pragma unroll
        for (int s = 0; s < 2 * UB; ++s) tmp[s] = hreg[s];
#pragma unroll
        for (int s = 0; s + 2 * UB < SL; ++s) hreg[s] = hreg[s + 2 * UB];
#pragma unroll
        for (int s = 0; s < 2 * UB; ++s) hreg[SL - 2 * UB + s] = tmp[s];
      }
    }
    if (valid) {
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const int j = 4 * s + t;
        if (j < r) {
          a.H[(long)j * a.ld + col] = hreg[s];
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

// ---- phase-convoy tensor-core sweep (default) --------------------------------
//
// Measured on B200 (tools/probe/contend_probe.cu, profiles/r01_notes.md): FP64
// scalar instructions share the FP64 pipe with DMMA, and a dependent DADD/DMUL
// waits ~16 cycles per DMMA-issuing warp on its SM sub-partition (8 -> 56
// cycles with three).  The row-by-row block solve is a chain of such ops, so
// interleaving it with other warps' DMMAs (all previous variants) stretches it
// ~5×.  Here all warps of the CTA move in lock-step phases separated by
// __syncthreads: every warp issues its block products (DMMA phase, pipe
// saturated), then every warp solves its block (scalar phase, pipe free).
// The solve chain is also shortened: the diagonal block's lower triangle
// (diagonal included) is zeroed in the DMMA operand, so
//     b_k = C_k - S_k - sum_{j<k in block} G_kj h_new_j
// needs one DMUL + one DFMA per row on the chain, and max(t, 0) is an integer
// compare (t > 0 exactly: 0 < bits(t) <= bits(+inf)).
ENMF_DEV double pos_part(double t) {
  const long long b = __double_as_longlong(t);
  return (b > 0 && b <= 0x7FF0000000000000LL) ? t : 0.0;
}

template <int RMAX>
constexpr int cv_smem_bytes() {
  return RMAX * (RMAX + 4) * 8 + 2 * RMAX * 8 + (RMAX / 8) * 72 * 8;
}

// MODE (timing experiments only): 0 = normal, 1 = skeleton without the row
// chain (wrong results), 2 = no phase barriers.
template <int RMAX, int UB, int NW, int MODE = 0>
__global__ void __launch_bounds__(NW * 32, 1) sweep_cv(Args a, int ntiles) {
  constexpr int LDG = RMAX + 4;
  constexpr int SL = RMAX / 4;
  constexpr int NB = RMAX / 8;
  constexpr int NTH = NW * 32;
  static_assert(NB % UB == 0, "row blocks per group");
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;                  // skewed G, diagonal blocks: strictly upper part only
  double* Gd = sm + RMAX * LDG;
  double* Gi = Gd + RMAX;
  double* GL = Gi + RMAX;           // [NB][8][9]: strictly lower part of each diagonal block
  __shared__ double red[NTH + 33];

  const int r = a.r;
  for (int e = threadIdx.x; e < RMAX * RMAX; e += NTH) {
    const int k = e / RMAX, c = e % RMAX;
    const int j = (c + 8 * (k / 8)) & (RMAX - 1);
    const double v = (k < r && j < r) ? a.G[(long)k * r + j] : 0.0;
    const bool diagblk = c < 8;      // rotated column c in [0, 8) <=> j in k's own block
    Gs[k * LDG + c] = (diagblk && c <= (k & 7)) ? 0.0 : v;
    if (diagblk) GL[(k >> 3) * 72 + (k & 7) * 9 + c] = (c < (k & 7)) ? v : 0.0;
  }
  for (int k = threadIdx.x; k < RMAX; k += NTH) {
    const double d = k < r ? a.G[(long)k * r + k] : 1.0;
    Gd[k] = d;
    Gi[k] = __ddiv_rn(1.0, d);
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  double gain = 0.0;
  int nf = 0;
  const int sg0 = g * 4 + ((2 * t) & 3), sg1 = g * 4 + ((2 * t + 1) & 3);
  const bool upper = t >= 2;
  const int ss_lo = g * 4 + (t >> 1), ss_hi = g * 4 + 2 + (t >> 1);
  const bool odd = t & 1;
  long long prof[6] = {0, 0, 0, 0, 0, 0};   // MODE 3: dmma, bar1, scalar, bar2, tile-load, total
  const long long tstart = (MODE == 3) ? clock64() : 0;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long col = ((long)tile * NW + warp) * 8 + g;
    const bool valid = col < a.N;
    long long tl0 = 0;
    if (MODE == 3) tl0 = clock64();
    double hreg[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      const int j = 4 * s + t;
      hreg[s] = (valid && j < r) ? src[(long)j * a.ld + col] : 0.0;
    }
    const double* cp = a.C + col;
    double cn0 = (valid && 2 * t < r) ? cp[(long)(2 * t) * a.ld] : 0.0;
    double cn1 = (valid && 2 * t + 1 < r) ? cp[(long)(2 * t + 1) * a.ld] : 0.0;
    if (MODE == 3) {
      if (hreg[SL - 1] == 12345.678 || cn1 == 0.123) gain += 1.0;
      prof[4] += clock64() - tl0;
    }
    const double* gbase = Gs + g * LDG + t;
#pragma unroll 1
    for (int q = 0; q < NB / UB; ++q) {
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int b = UB * q + u;
        const int k0 = 8 * b;
        const int ka = k0 + 2 * t;
        const double cc0 = cn0, cc1 = cn1;
        if (b + 1 < NB) {
          cn0 = (valid && ka + 8 < r) ? cp[(long)(ka + 8) * a.ld] : 0.0;
          cn1 = (valid && ka + 9 < r) ? cp[(long)(ka + 9) * a.ld] : 0.0;
        }
        long long tk0 = 0;
        if (MODE == 3) tk0 = clock64();
        // ---- DMMA phase ----
        double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        const double* gb = gbase + k0 * LDG;
#pragma unroll
        for (int s = 0; s < SL; ++s) {
          const int c = (4 * s - 8 * u + RMAX) & (RMAX - 1);
          dmma884(acc[s & 3][0], acc[s & 3][1], hreg[s], gb[c]);
        }
        const double S0 = __dadd_rn(__dadd_rn(acc[0][0], acc[1][0]), __dadd_rn(acc[2][0], acc[3][0]));
        const double S1 = __dadd_rn(__dadd_rn(acc[0][1], acc[1][1]), __dadd_rn(acc[2][1], acc[3][1]));
        if (MODE == 3) {
          // force completion of the products before reading the clock
          if (S0 == 12345.678 && S1 == 0.5) gain += 1.0;
          prof[0] += clock64() - tk0;
        }
        const double xa0 = __shfl_sync(0xffffffffu, hreg[2 * u], sg0);
        const double xb0 = __shfl_sync(0xffffffffu, hreg[2 * u + 1], sg0);
        const double xa1 = __shfl_sync(0xffffffffu, hreg[2 * u], sg1);
        const double xb1 = __shfl_sync(0xffffffffu, hreg[2 * u + 1], sg1);
        const double x0 = upper ? xb0 : xa0, x1 = upper ? xb1 : xa1;
        double b0 = __dsub_rn(cc0, S0);
        double b1 = __dsub_rn(cc1, S1);
        const double* gl0 = GL + b * 72 + (2 * t) * 9;
        const double* gl1 = gl0 + 9;
        const double i00 = Gi[ka], i11 = Gi[ka + 1];
        const double l10 = gl1[2 * t];    // G[ka+1][ka]
        long long tk1 = 0;
        if (MODE == 3) tk1 = clock64();
        if (MODE != 2) __syncthreads();
        long long tk2 = 0;
        if (MODE == 3) {
          tk2 = clock64();
          prof[1] += tk2 - tk1;
        }
        // ---- scalar phase: rows k0..k0+7 in order, row k0+i in lane t = i/2 ----
        double t0 = 0.0, t1 = 0.0, h0 = 0.0, h1 = 0.0;
        if (MODE == 1) {
          t0 = __dmul_rn(b0, i00); h0 = pos_part(t0);
          t1 = __dmul_rn(b1, i11); h1 = pos_part(t1);
        }
#pragma unroll
        for (int i = 0; i < (MODE == 1 ? 0 : 8); i += 2) {
          const double tt0 = __dmul_rn(b0, i00);
          const double hh0 = pos_part(tt0);
          const double tt1 = __dmul_rn(fma(-l10, hh0, b1), i11);
          const double hh1 = pos_part(tt1);
          if (2 * t == i) {
            t0 = tt0; h0 = hh0; t1 = tt1; h1 = hh1;
          }
          if (i < 6) {
            const double e0 = __shfl_sync(0xffffffffu, hh0, g * 4 + i / 2);
            const double e1 = __shfl_sync(0xffffffffu, hh1, g * 4 + i / 2);
            if (2 * t > i) {
              b0 = fma(-gl0[i], e0, b0);
              b1 = fma(-gl1[i], e0, b1);
              b0 = fma(-gl0[i + 1], e1, b0);
              b1 = fma(-gl1[i + 1], e1, b1);
            }
          }
        }
        {
          const double g00 = Gd[ka], g11 = Gd[ka + 1];
          const double o0 = __dsub_rn(x0, t0), n0 = __dsub_rn(h0, t0);
          const double o1 = __dsub_rn(x1, t1), n1 = __dsub_rn(h1, t1);
          gain = fma(g00, __dsub_rn(__dmul_rn(o0, o0), __dmul_rn(n0, n0)), gain);
          gain = fma(g11, __dsub_rn(__dmul_rn(o1, o1), __dmul_rn(n1, n1)), gain);
        }
        const double y0 = __shfl_sync(0xffffffffu, h0, ss_lo);
        const double y1 = __shfl_sync(0xffffffffu, h1, ss_lo);
        const double z0 = __shfl_sync(0xffffffffu, h0, ss_hi);
        const double z1 = __shfl_sync(0xffffffffu, h1, ss_hi);
        hreg[2 * u] = odd ? y1 : y0;
        hreg[2 * u + 1] = odd ? z1 : z0;
        long long tk3 = 0;
        if (MODE == 3) {
          if (hreg[2 * u] == 12345.678) gain += 1.0;
          tk3 = clock64();
          prof[2] += tk3 - tk2;
        }
        if (MODE != 2) __syncthreads();
        if (MODE == 3) prof[3] += clock64() - tk3;
      }
      if (NB / UB > 1) {
        double tmp[2 * UB];
#pragma unroll
        for (int s = 0; s < 2 * UB; ++s) tmp[s] = hreg[s];
#pragma unroll
        for (int s = 0; s + 2 * UB < SL; ++s) hreg[s] = hreg[s + 2 * UB];
#pragma unroll
        for (int s = 0; s < 2 * UB; ++s) hreg[SL - 2 * UB + s] = tmp[s];
      }
    }
    if (valid) {
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const int j = 4 * s + t;
        if (j < r) {
          a.H[(long)j * a.ld + col] = hreg[s];
          nf |= !isfinite(hreg[s]);
        }
      }
    }
  }
  if (MODE == 3 && lane == 0 && a.terms) {
    prof[5] = clock64() - tstart;
    double* o = a.terms + ((long)blockIdx.x * NW + warp) * 8;
    for (int i = 0; i < 6; ++i) o[i] = (double)prof[i];
  }
  const double bg = block_reduce_sum_any(gain, red);
  nf = __syncthreads_or(nf);
  last_block_reduce_n<NTH>(a, bg, nf, red);
}

// ---- look-ahead tensor-core sweep ---------------------------------------------
//
// Left-looking blocked Gauss-Seidel (sweep_dmma_t layout: lane (g, t) owns rows
// k0+2t, k0+2t+1 of column g in the block being solved) with a one-block
// look-ahead: while block b is solved row by row (latency-bound), the warp
// already issues the 30 DMMAs of block b+1's products with every row block
// except b,
//     P_{b+1} = sum_{j not in block b} G[b+1 rows][j] · h_j,
// which do not depend on block b's solution; block b+1 then only adds the two
// DMMAs of G[b+1 rows][block b] · H_new[b].  The solve and the next block's
// tensor work are independent instruction streams in one basic block, so the
// scheduler interleaves them and the sequential chain hides behind DMMA issue.
template <int RMAX, int NW>
__global__ void __launch_bounds__(NW * 32, 1) sweep_la(Args a, int ntiles) {
  constexpr int LDG = RMAX + 4;
  constexpr int SL = RMAX / 4;
  constexpr int NB = RMAX / 8;
  constexpr int NTH = NW * 32;
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;
  double* Gd = sm + RMAX * LDG;
  double* Gi = Gd + RMAX;
  __shared__ double red[NTH + 33];

  const int r = a.r;
  {
    // Gs[k][c] = G[k][(c + 8·(k/8)) mod RMAX], zero padding (see sweep_dmma_p)
    constexpr int CH = RMAX / 2;
    const bool vec = (r % 2 == 0) && (((uintptr_t)a.G & 15) == 0);
    for (int e = threadIdx.x; e < RMAX * CH; e += NTH) {
      const int k = e / CH, c = (e % CH) * 2;
      const int j = (c + 8 * (k / 8)) & (RMAX - 1);
      const unsigned dst = (unsigned)__cvta_generic_to_shared(Gs + k * LDG + c);
      if (vec) {
        const int valid = (k < r && j < r) ? 16 : 0;
        const double* srcp = valid ? a.G + (long)k * r + j : a.G;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(srcp), "r"(valid));
      } else {
        Gs[k * LDG + c] = (k < r && j < r) ? a.G[(long)k * r + j] : 0.0;
        Gs[k * LDG + c + 1] = (k < r && j + 1 < r) ? a.G[(long)k * r + j + 1] : 0.0;
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
  const int sg0 = g * 4 + ((2 * t) & 3), sg1 = g * 4 + ((2 * t + 1) & 3);
  const bool upper = t >= 2;
  const int ss_lo = g * 4 + (t >> 1), ss_hi = g * 4 + 2 + (t >> 1);
  const bool odd = t & 1;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long col = ((long)tile * NW + warp) * 8 + g;
    const bool valid = col < a.N;
    double hreg[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      const int j = 4 * s + t;
      hreg[s] = (valid && j < r) ? src[(long)j * a.ld + col] : 0.0;
    }
    const double* cp = a.C + col;
    double cn0 = (valid && 2 * t < r) ? cp[(long)(2 * t) * a.ld] : 0.0;
    double cn1 = (valid && 2 * t + 1 < r) ? cp[(long)(2 * t + 1) * a.ld] : 0.0;
    if (first) {
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
      first = false;
    }
    const double* gbase = Gs + g * LDG + t;
    // P for block 0: all slots (block 0's rows are old values)
    double pa[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int s = 0; s < SL; ++s) dmma884(pa[s & 3][0], pa[s & 3][1], hreg[s], gbase[4 * s]);
#pragma unroll 1
    for (int b = 0; b < NB; ++b) {
      const int k0 = 8 * b;
      const int ka = k0 + 2 * t;
      const double cc0 = cn0, cc1 = cn1;
      if (b + 1 < NB) {
        cn0 = (valid && ka + 8 < r) ? cp[(long)(ka + 8) * a.ld] : 0.0;
        cn1 = (valid && ka + 9 < r) ? cp[(long)(ka + 9) * a.ld] : 0.0;
      }
      const double* gb = gbase + k0 * LDG;
      // complete S_b with the previous block's new rows (slots SL-2, SL-1)
      double S0 = __dadd_rn(__dadd_rn(pa[0][0], pa[1][0]), __dadd_rn(pa[2][0], pa[3][0]));
      double S1 = __dadd_rn(__dadd_rn(pa[0][1], pa[1][1]), __dadd_rn(pa[2][1], pa[3][1]));
      if (b > 0) {
        dmma884(S0, S1, hreg[SL - 2], gb[4 * (SL - 2)]);
        dmma884(S0, S1, hreg[SL - 1], gb[4 * (SL - 1)]);
      }
      // look-ahead: P_{b+1} over all slots except this block's (0, 1), issued in
      // five chunks interleaved with the solve below (in-order issue per warp)
#pragma unroll
      for (int i = 0; i < 4; ++i) pa[i][0] = pa[i][1] = 0.0;
      const bool ahead = b + 1 < NB;
      const double* gn = gb + 8 * LDG;
      constexpr int CHK = (SL - 2 + 4) / 5;   // DMMAs per chunk
      auto look = [&](int chunk) {
        if (ahead) {
#pragma unroll
          for (int q = 0; q < CHK; ++q) {
            const int s = 2 + chunk * CHK + q;
            if (s < SL) dmma884(pa[s & 3][0], pa[s & 3][1], hreg[s], gn[4 * s - 8]);
          }
        }
      };
      look(0);
      // solve block b
      const double xa0 = __shfl_sync(0xffffffffu, hreg[0], sg0);
      const double xb0 = __shfl_sync(0xffffffffu, hreg[1], sg0);
      const double xa1 = __shfl_sync(0xffffffffu, hreg[0], sg1);
      const double xb1 = __shfl_sync(0xffffffffu, hreg[1], sg1);
      const double x0 = upper ? xb0 : xa0, x1 = upper ? xb1 : xa1;
      const double* gk0 = Gs + ka * LDG;
      const double* gk1 = gk0 + LDG;
      const double g00 = Gd[ka], g11 = Gd[ka + 1];
      const double i00 = Gi[ka], i11 = Gi[ka + 1];
      double b0 = fma(g00, x0, __dsub_rn(cc0, S0));
      double b1 = fma(g11, x1, __dsub_rn(cc1, S1));
      double h0 = x0, h1 = x1, t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        // branch-free: every lane computes, only the owner's values are kept
        const bool own = 2 * t == i;
        const double tt0 = __dmul_rn(b0, i00);
        const double hh0 = tt0 > 0.0 ? tt0 : 0.0;
        const double dd0 = __dsub_rn(hh0, x0);
        const double bb1 = fma(-gk1[i], dd0, b1);
        const double tt1 = __dmul_rn(bb1, i11);
        const double hh1 = tt1 > 0.0 ? tt1 : 0.0;
        const double dd1 = __dsub_rn(hh1, x1);
        if (own) {
          t0 = tt0; h0 = hh0; t1 = tt1; h1 = hh1;
        }
        look(1 + i / 2);
        if (i < 6) {
          const double e0 = __shfl_sync(0xffffffffu, dd0, g * 4 + i / 2);
          const double e1 = __shfl_sync(0xffffffffu, dd1, g * 4 + i / 2);
          if (2 * t > i) {
            b0 = fma(-gk0[i], e0, b0);
            b0 = fma(-gk0[i + 1], e1, b0);
            b1 = fma(-gk1[i], e0, b1);
            b1 = fma(-gk1[i + 1], e1, b1);
          }
        }
      }
      {
        const double o0 = __dsub_rn(x0, t0), n0 = __dsub_rn(h0, t0);
        const double o1 = __dsub_rn(x1, t1), n1 = __dsub_rn(h1, t1);
        gain = fma(g00, __dsub_rn(__dmul_rn(o0, o0), __dmul_rn(n0, n0)), gain);
        gain = fma(g11, __dsub_rn(__dmul_rn(o1, o1), __dmul_rn(n1, n1)), gain);
      }
      const double y0 = __shfl_sync(0xffffffffu, h0, ss_lo);
      const double y1 = __shfl_sync(0xffffffffu, h1, ss_lo);
      const double z0 = __shfl_sync(0xffffffffu, h0, ss_hi);
      const double z1 = __shfl_sync(0xffffffffu, h1, ss_hi);
      // rotate by two slots; this block's new rows go to SL-2, SL-1
#pragma unroll
      for (int s = 0; s + 2 < SL; ++s) hreg[s] = hreg[s + 2];
      hreg[SL - 2] = odd ? y1 : y0;
      hreg[SL - 1] = odd ? z1 : z0;
    }
    if (valid) {
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const int j = 4 * s + t;
        if (j < r) {
          a.H[(long)j * a.ld + col] = hreg[s];
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

// ---- right-looking tensor-core sweep ------------------------------------------
//
// Gauss-Seidel written right-looking.  Per column keep the residual
//     R_k = C_k - sum_{j processed} G_kj h_new_j - sum_{j not yet processed, j != k} G_kj h_old_j
// so that row k's update is  h_new_k = max(0, R_k / G_kk)  (nnls.hpp:116-134).
// For a tile of 8 columns per warp (lane (g, t): column g, rows 8K+2t, 8K+2t+1
// of every 8-row block K — 32 doubles of R in registers):
//   1. R = C - U·H_old, U = the strictly upper part of G (block-upper tiles plus
//      the strictly upper triangle of each diagonal 8×8 block): independent DMMA
//      chains, one per row block.
//   2. for each row block b: finish its 8 rows sequentially (lower triangle of
//      the diagonal block, shuffles inside the column's lane quad), write them,
//      then R[K'] -= G[K', b]·H_new[b] for every later block K' > b (DMMA).
// The DMMA work equals the reference's r² per column; unlike the left-looking
// kernels each block's products are independent of the block solve that
// follows, so other warps' tensor work overlaps it.  -G is staged in shared
// memory so every DMMA accumulates (D = A·B + C) straight into R.
template <int RMAX>
constexpr int rl_smem_bytes() {
  return RMAX * (RMAX + 4) * 8 + 2 * RMAX * 8 + (RMAX / 8) * 64 * 8;
}

template <int RMAX, int NW>
__global__ void __launch_bounds__(NW * 32, 1) sweep_rl(Args a, int ntiles) {
  constexpr int LDG = RMAX + 4;
  constexpr int NB = RMAX / 8;
  constexpr int NTH = NW * 32;
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gn = sm;                  // -G, full (diagonal blocks: strictly upper part only, rest 0)
  double* Gd = sm + RMAX * LDG;     // G_kk (1 on padding rows)
  double* Gi = Gd + RMAX;           // 1 / G_kk
  double* GL = Gi + RMAX;           // [NB][8][8] +G strictly lower part of each diagonal block
  __shared__ double red[NTH + 33];

  const int r = a.r;
  for (int e = threadIdx.x; e < RMAX * RMAX; e += NTH) {
    const int k = e / RMAX, j = e % RMAX;
    const double v = (k < r && j < r) ? a.G[(long)k * r + j] : 0.0;
    const bool same = (k >> 3) == (j >> 3);
    Gn[k * LDG + j] = (!same || j > k) ? -v : 0.0;
    if (same) GL[(k >> 3) * 64 + (k & 7) * 8 + (j & 7)] = (j < k) ? v : 0.0;
  }
  for (int k = threadIdx.x; k < RMAX; k += NTH) {
    const double d = k < r ? a.G[(long)k * r + k] : 1.0;
    Gd[k] = d;
    Gi[k] = __ddiv_rn(1.0, d);
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  const int ss_lo = g * 4 + (t >> 1), ss_hi = g * 4 + 2 + (t >> 1);
  const bool odd = t & 1;
  double gain = 0.0;
  int nf = 0;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long col = ((long)tile * NW + warp) * 8 + g;
    const bool valid = col < a.N;
    const double* hs = src + col;
    double* ho = a.H + col;
    const double* cs = a.C + col;
    auto ld = [&](const double* p, int row) -> double {
      return (valid && row < r) ? p[(long)row * a.ld] : 0.0;
    };
    // ---- phase 1: R = C - U·H_old --------------------------------------------
    double R[NB][2];
#pragma unroll
    for (int K = 0; K < NB; ++K) {
      R[K][0] = ld(cs, 8 * K + 2 * t);
      R[K][1] = ld(cs, 8 * K + 2 * t + 1);
    }
#pragma unroll
    for (int jb = 0; jb < NB; ++jb) {
      const double a0 = ld(hs, 8 * jb + t), a1 = ld(hs, 8 * jb + 4 + t);
      const double* gcol = Gn + g * LDG + 8 * jb + t;
#pragma unroll
      for (int K = 0; K <= jb; ++K) {   // K == jb: strictly upper triangle of the diagonal block
        dmma884(R[K][0], R[K][1], a0, gcol[8 * K * LDG]);
        dmma884(R[K][0], R[K][1], a1, gcol[8 * K * LDG + 4]);
      }
    }
    // ---- phase 2: block solves + right-looking updates -------------------------
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int ka = 8 * b + 2 * t;
      const double x0 = ld(hs, ka), x1 = ld(hs, ka + 1);
      const double* gl0 = GL + b * 64 + (2 * t) * 8;   // row ka of the diagonal block (lower part)
      const double* gl1 = gl0 + 8;                     // row ka+1
      const double i0 = Gi[ka], i1 = Gi[ka + 1];
      double b0 = R[b][0], b1 = R[b][1];
      double h0 = 0.0, h1 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        if (2 * t == i) {
          t0 = __dmul_rn(b0, i0);
          h0 = t0 > 0.0 ? t0 : 0.0;
          b1 = fma(-gl1[i], h0, b1);
          t1 = __dmul_rn(b1, i1);
          h1 = t1 > 0.0 ? t1 : 0.0;
        }
        if (i < 6) {
          const double e0 = __shfl_sync(0xffffffffu, h0, g * 4 + i / 2);
          const double e1 = __shfl_sync(0xffffffffu, h1, g * 4 + i / 2);
          if (2 * t > i) {
            b0 = fma(-gl0[i], e0, b0);
            b0 = fma(-gl0[i + 1], e1, b0);
            b1 = fma(-gl1[i], e0, b1);
            b1 = fma(-gl1[i + 1], e1, b1);
          }
        }
      }
      {
        const double g0 = Gd[ka], g1 = Gd[ka + 1];
        const double o0 = __dsub_rn(x0, t0), n0 = __dsub_rn(h0, t0);
        const double o1 = __dsub_rn(x1, t1), n1 = __dsub_rn(h1, t1);
        gain = fma(g0, __dsub_rn(__dmul_rn(o0, o0), __dmul_rn(n0, n0)), gain);
        gain = fma(g1, __dsub_rn(__dmul_rn(o1, o1), __dmul_rn(n1, n1)), gain);
      }
      if (valid) {
        if (ka < r) ho[(long)ka * a.ld] = h0;
        if (ka + 1 < r) ho[(long)(ka + 1) * a.ld] = h1;
        nf |= !isfinite(h0) | !isfinite(h1);
      }
      if (b + 1 < NB) {
        // A fragments of H_new[b]: rows 8b+t and 8b+4+t of column g
        const double y0 = __shfl_sync(0xffffffffu, h0, ss_lo);
        const double y1 = __shfl_sync(0xffffffffu, h1, ss_lo);
        const double z0 = __shfl_sync(0xffffffffu, h0, ss_hi);
        const double z1 = __shfl_sync(0xffffffffu, h1, ss_hi);
        const double a0 = odd ? y1 : y0, a1 = odd ? z1 : z0;
        const double* gcol = Gn + g * LDG + 8 * b + t;
#pragma unroll
        for (int K = b + 1; K < NB; ++K) {
          dmma884(R[K][0], R[K][1], a0, gcol[8 * K * LDG]);
          dmma884(R[K][0], R[K][1], a1, gcol[8 * K * LDG + 4]);
        }
      }
    }
  }
  const double bg = block_reduce_sum_any(gain, red);
  nf = __syncthreads_or(nf);
  last_block_reduce_n<NTH>(a, bg, nf, red);
}

// ---- paired-warp tensor-core sweep (default) ----------------------------------
//
// Every SM sub-partition runs one PAIR of warps over its own 32 columns:
//   * the product warp issues the DMMAs of the block products
//         S_b = G[b-rows, :] · H        (A = Gram fragment in registers, B = H in smem)
//   * the row warp owns one column per lane and finishes the 8 rows of block b
//     sequentially (nnls.hpp:117-148 per row), entirely in registers, writing the
//     new rows straight into the H tile.
// The two phases strictly alternate (named-barrier hand-offs, bar.arrive by the
// producer of a tile, bar.sync by its consumer): measured on B200
// (tools/probe/pipe_probe.cu, profiles/r01_latency_probes.txt), scalar FP64
// instructions on a sub-partition whose DMMA pipe is streaming are starved
// (~75 cycles per independent op, ~500 per dependent op), so the row chain runs
// while the sub-partition's DMMA pipe is idle and takes ~0.3 K cycles instead of
// ~1.7 K when overlapped.  Diagonal blocks enter the DMMA with their lower triangle
// (diagonal included) zeroed, so the row warp only subtracts
// sum_{j<k in block} G_kj h_new_j.
//
// Gram fragments come pre-arranged by ws_prep (once per inner solve): Gf holds,
// for row block b and k-step pair s2, the two A-fragment values of every lane
// contiguously, so a lane fetches two k-steps with one 16-byte load, and the
// fragments of block b+1 stream into the registers freed by block b.  The H tile
// is stored with 16-byte chunks holding columns (c, c+8) and an XOR swizzle per
// row, so each lane reads the B fragments of its 4 column tiles with two
// conflict-free 16-byte loads per k-step.
constexpr int WS_SLD = 40;   // S tile row stride: conflict-free 16-byte fragment stores

template <int RMAX>
constexpr int ws_smem_bytes() {
  return (4 * (RMAX * 32 + 8 * WS_SLD) + (RMAX / 8) * 48) * 8;
}

// position of (row k, column c) in a swizzled 32-column tile
ENMF_DEV int ws_pos(int k, int c) {
  const int sw = ((k & 1) << 2) | ((k >> 1) & 1);
  return k * 32 + 2 * ((2 * (c & 7) + (c >> 4)) ^ sw) + ((c >> 3) & 1);
}

ENMF_DEV void nb_sync(int id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory"); }
// clock64 after a shared-memory load that the hardware cannot issue before the preceding
// barrier resolves (bar.sync defers its blocking; timing experiments only)
ENMF_DEV long long clock_after_smem(const double* p) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];\n" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
  long long t;
  asm volatile("{ .reg .pred q; setp.eq.f64 q, %1, %1; mov.u64 %0, %%clock64; }\n" : "=l"(t) : "d"(v) : "memory");
  return t;
}
ENMF_DEV void nb_arrive(int id) { asm volatile("bar.arrive %0, 64;\n" ::"r"(id) : "memory"); }

ENMF_DEV double pos_part_ws(double t) {
  const long long b = __double_as_longlong(t);
  return (b > 0 && b <= 0x7FF0000000000000LL) ? t : 0.0;   // t > 0 (NaN -> 0, as `t > 0 ? t : 0`)
}

// Gf[((b·KS/2 + s2)·32 + lane)·2 + e] = G[8b + lane/4][4(2·s2+e) + lane%4], zero outside r×r,
// on/below the diagonal inside diagonal blocks, and — for odd b — in the columns of block
// b-1, whose fragments go to Gf[RMAX² + ...] instead (the "tail" of the paired product).
template <int RMAX>
__global__ void ws_prep(const double* G, int r, double* Gf, const DevState* st, const HalsCtl* ctl) {
  if ((st && !dev_active(st)) || !ctl->cont) return;
  constexpr int KS = RMAX / 4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < RMAX * RMAX; i += gridDim.x * blockDim.x) {
    const int e = i & 1, lane = (i >> 1) & 31, s2 = (i >> 6) % (KS / 2), b = (i >> 6) / (KS / 2);
    const int s = 2 * s2 + e, gi = lane >> 2, gt = lane & 3;
    const int row = 8 * b + gi, col = 4 * s + gt;
    double v = 0.0;
    if (row < r && col < r && !((s >> 1) == b && col - 8 * b <= gi)) v = G[(long)row * r + col];
    const bool tail = (b & 1) && s2 == b - 1;
    Gf[i] = tail ? 0.0 : v;
    if (tail) Gf[RMAX * RMAX + (b >> 1) * 64 + lane * 2 + e] = v;
  }
}

// B fragments of k-steps (2j, 2j+1) — rows 8j..8j+7 — for the NT column tiles of a pair
template <int NT>
ENMF_DEV void ws_ldb(const double* Hs, int j, int gt, int bx0, int bx1, double2 (&p)[4]) {
  const int k0 = 8 * j + gt, k1 = k0 + 4;
  p[0] = *reinterpret_cast<const double2*>(Hs + k0 * 32 + bx0);
  if (NT > 2) p[1] = *reinterpret_cast<const double2*>(Hs + k0 * 32 + bx1);
  p[2] = *reinterpret_cast<const double2*>(Hs + k1 * 32 + bx0);
  if (NT > 2) p[3] = *reinterpret_cast<const double2*>(Hs + k1 * 32 + bx1);
}

// acc[t] += a0 · B(k-step 2j) + a1 · B(k-step 2j+1) for the NT tiles
template <int NT>
ENMF_DEV void ws_mma2(double (&acc)[4][2], double a0, double a1, const double2 (&p)[4]) {
  dmma884(acc[0][0], acc[0][1], a0, p[0].x);
  if (NT > 1) dmma884(acc[1][0], acc[1][1], a0, p[0].y);
  if (NT > 2) dmma884(acc[2][0], acc[2][1], a0, p[1].x);
  if (NT > 3) dmma884(acc[3][0], acc[3][1], a0, p[1].y);
  dmma884(acc[0][0], acc[0][1], a1, p[2].x);
  if (NT > 1) dmma884(acc[1][0], acc[1][1], a1, p[2].y);
  if (NT > 2) dmma884(acc[2][0], acc[2][1], a1, p[3].x);
  if (NT > 3) dmma884(acc[3][0], acc[3][1], a1, p[3].y);
}

ENMF_DEV void ws_store_s(double* Ss, int gi, int gt, const double (&acc)[4][2]) {
#pragma unroll
  for (int t = 0; t < 4; ++t)
    *reinterpret_cast<double2*>(Ss + gi * WS_SLD + t * 8 + 2 * gt) = make_double2(acc[t][0], acc[t][1]);
}

// The product warp's part of one round: row blocks in pairs (b, b+1).  One pass
// over the H tile feeds both products — S_b over every row block and S_{b+1}
// over every block but b — so each B fragment is loaded once for two A
// fragments; S_{b+1} then gets block b's new rows (its "tail") once the row warp
// has solved block b.  The Gram fragments of the next pair are fetched while the
// row warp works (DMMA pipe idle).
template <int KS, int NB, int NT, bool PROF, int SKIP>
ENMF_DEV void ws_producer_round(const double* Hs, double* Ss, const double2* gf, int gi, int gt, int bx0, int bx1,
                                int idS, int idH, long long* pw) {
  double A0[KS], A1[KS];
#pragma unroll
  for (int s = 0; s < KS; s += 2) {
    const double2 f0 = gf[(s / 2) * 32];
    const double2 f1 = gf[(KS / 2 + s / 2) * 32];
    A0[s] = f0.x; A0[s + 1] = f0.y;
    A1[s] = f1.x; A1[s + 1] = f1.y;
  }
#pragma unroll 1
  for (int b = 0; b < NB; b += 2) {
    const long long c0 = PROF ? clock64() : 0;
    if (b > 0) nb_sync(idH);                // rows of block b-1 are final in the tile
    const long long c1 = PROF ? clock_after_smem(Ss) : 0;
    if (PROF) pw[0] += c1 - c0;
    double acc0[4][2], acc1[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) acc0[t][0] = acc0[t][1] = acc1[t][0] = acc1[t][1] = 0.0;
    if (!(SKIP & 2)) {
#pragma unroll
      for (int j = 0; j < KS / 2; ++j) {   // (block b's fragments of A1 are zero: see ws_prep)
        double2 p[4];
        ws_ldb<NT>(Hs, j, gt, bx0, bx1, p);
        ws_mma2<NT>(acc0, A0[2 * j], A0[2 * j + 1], p);
        ws_mma2<NT>(acc1, A1[2 * j], A1[2 * j + 1], p);
      }
    }
    ws_store_s(Ss, gi, gt, acc0);
    nb_arrive(idS);                          // S_b ready: the row warp solves block b
    if (PROF) pw[2] += clock64() - c1;
    // while it does: this pair's tail fragments and the next pair's Gram fragments
    const double2 tl = gf[(16 * KS * KS + (b >> 1) * 64) / 2];   // Gf tails (ws_prep)
    if (b + 2 < NB) {
#pragma unroll
      for (int s = 0; s < KS; s += 2) {
        const double2 f0 = gf[(((b + 2) * KS / 2) + s / 2) * 32];
        const double2 f1 = gf[(((b + 3) * KS / 2) + s / 2) * 32];
        A0[s] = f0.x; A0[s + 1] = f0.y;
        A1[s] = f1.x; A1[s + 1] = f1.y;
      }
    }
    const long long c3 = PROF ? clock64() : 0;
    nb_sync(idH);                            // block b solved
    const long long c2 = PROF ? clock_after_smem(Ss) : 0;
    if (PROF) pw[0] += c2 - c3;
    if (!(SKIP & 2)) {
      double2 p[4];
      ws_ldb<NT>(Hs, b, gt, bx0, bx1, p);
      ws_mma2<NT>(acc1, tl.x, tl.y, p);
    }
    ws_store_s(Ss, gi, gt, acc1);
    nb_arrive(idS);                          // S_{b+1} ready
    if (PROF) pw[2] += clock64() - c2;
  }
}

// PROF (timing experiment): per-warp cycles [barrier wait, tile load, total, DMMA / row phase] into a.terms;
// SKIP (timing experiment, wrong results): 1 = row warps skip the row pass, 2 = product warps skip the DMMAs
// PERSIST: one launch runs every sweep of the solve.  Between sweeps the CTAs
// meet at a grid-wide decision point (the last CTA to arrive sums the per-CTA
// gains in fixed order, applies the stall rule — after the cross-GPU gain
// exchange when sharded — and publishes it through ctl->epoch), and the rounds
// alternate direction so the tile a pair finished a sweep with is the one it
// starts the next sweep with, already in shared memory.  Requires all CTAs to be
// co-resident (cooperative launch, one CTA per SM).
template <int RMAX, bool PROF = false, int SKIP = 0, bool PERSIST = false>
__global__ void __launch_bounds__(256, 1) sweep_ws(Args a, long ntiles) {
  constexpr int NB = RMAX / 8;
  constexpr int KS = RMAX / 4;
  const long long tk0 = PROF ? clock64() : 0;
  long long pw[4] = {0, 0, 0, 0};
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[256 + 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp & 3;
  const bool producer = warp < 4;
  double* Hs = sm + pair * (RMAX * 32);
  double* Ss = sm + 4 * RMAX * 32 + pair * 8 * WS_SLD;
  // per row block: lower triangle G[8b+l][8b+i] (i < l) at l(l-1)/2 + i, G_kk/2 at 28 + l,
  // 1/G_kk at 36 + l (padding rows: unit diagonal)
  double* Gc = sm + 4 * (RMAX * 32 + 8 * WS_SLD);
  const int r = a.r;
  for (int e = threadIdx.x; e < NB * 48; e += 256) {
    const int b = e / 48, j = e % 48;
    double v = 0.0;
    if (j < 28) {
      int l = 1;
      while (l * (l + 1) / 2 <= j) ++l;
      const int i = j - l * (l - 1) / 2, k = 8 * b + l, c = 8 * b + i;
      v = (k < r && c < r) ? a.G[(long)k * r + c] : 0.0;
    } else if (j < 44) {
      const int k = 8 * b + ((j - 28) & 7);
      const double d = k < r ? a.G[(long)k * r + k] : 1.0;
      v = j < 36 ? __dmul_rn(0.5, d) : __ddiv_rn(1.0, d);
    }
    Gc[e] = v;
  }
  __syncthreads();

  const int idS = 1 + pair, idH = 5 + pair, idP = 9 + pair;
  const long P = (long)gridDim.x * 4, q = (long)blockIdx.x * 4 + pair;
  const long tq0 = q * ntiles / P, cnt = (q + 1) * ntiles / P - tq0;
  const int rounds = (int)((cnt + 3) / 4);
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  double gain = 0.0;
  int nf = 0;
  __shared__ int s_flag;
  double first_total = 0.0;                 // persistent: the first sweep's total gain (stall rule)
  const int gi = lane >> 2, gt = lane & 3;
  // this lane's two 16-byte B-fragment chunks (tiles 0,1 and 2,3) within a row k with k & 3 == gt
  const int swz = ((gt & 1) << 2) | (gt >> 1);
  const int bx0 = 2 * ((2 * gi) ^ swz), bx1 = 2 * ((2 * gi + 1) ^ swz);
  const double2* gf = reinterpret_cast<const double2*>(a.Gf) + lane;
  int hoff[4];                              // swizzled position of column `lane` in a row k, by k & 3
#pragma unroll
  for (int j = 0; j < 4; ++j) hoff[j] = ws_pos(j, lane) - j * 32;

  for (int sw = 0;; ++sw) {
  for (int i = 0; i < rounds; ++i) {
    const int rd = (PERSIST && (sw & 1)) ? rounds - 1 - i : i;
    const long ta = tq0 + (long)rd * cnt / rounds;
    const int nt = (int)(tq0 + (long)(rd + 1) * cnt / rounds - ta);
    const long col0 = ta * 8;
    const long long tl0 = PROF ? clock64() : 0;
    // stage this round's 32 columns of H (zero outside r × N and past nt tiles);
    // persistent: the first round of a later sweep is still in shared memory
    nb_sync(idP);                           // previous round done with the tiles
    if (!(PERSIST && sw > 0 && i == 0)) {
      const int c = lane;
      const long col = col0 + c;
      const bool okc = c < nt * 8 && col < a.N;
      const double* sp = src + col;
      for (int k = producer ? 0 : 1; k < RMAX; k += 2) {
        const bool ok = okc && k < r;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(Hs + ws_pos(k, c));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst),
                     "l"(ok ? sp + (long)k * a.ld : src), "r"(ok ? 8 : 0));
      }
      asm volatile("cp.async.wait_all;\n" ::);
    }
    nb_sync(idP);
    if (PROF) pw[1] += clock64() - tl0;

    if (producer) {
      switch (nt) {
        case 4: ws_producer_round<KS, NB, 4, PROF, SKIP>(Hs, Ss, gf, gi, gt, bx0, bx1, idS, idH, pw); break;
        case 3: ws_producer_round<KS, NB, 3, PROF, SKIP>(Hs, Ss, gf, gi, gt, bx0, bx1, idS, idH, pw); break;
        case 2: ws_producer_round<KS, NB, 2, PROF, SKIP>(Hs, Ss, gf, gi, gt, bx0, bx1, idS, idH, pw); break;
        default: ws_producer_round<KS, NB, 1, PROF, SKIP>(Hs, Ss, gf, gi, gt, bx0, bx1, idS, idH, pw); break;
      }
    } else {
      const long col = col0 + lane;
      const bool valid = lane < nt * 8 && col < a.N;
      const int rv = valid ? r : 0;         // rows this lane loads / stores
      const double* cp = a.C + col;
      double* hp = a.H + col;
      double cn[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) cn[i] = i < rv ? cp[(long)i * a.ld] : 0.0;
      long long hmax = 0;                   // largest bit pattern stored (h >= 0: +inf is the only non-finite)
#pragma unroll 1
      for (int b = 0; b < NB; ++b) {
        double bb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) bb[i] = cn[i];
        if (b + 1 < NB) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int k = 8 * (b + 1) + i;
            cn[i] = k < rv ? cp[(long)k * a.ld] : 0.0;
          }
        }
        // this block's lower triangle, half diagonal and inverse diagonal (broadcast loads)
        double gc[48];
        {
          const double2* gb = reinterpret_cast<const double2*>(Gc + b * 48);
#pragma unroll
          for (int j = 0; j < 22; ++j) {
            const double2 v = gb[j];
            gc[2 * j] = v.x;
            gc[2 * j + 1] = v.y;
          }
        }
        const long long c0 = PROF ? clock64() : 0;
        nb_sync(idS);
        const long long c1 = PROF ? clock_after_smem(Ss + lane) : 0;
        if (PROF) pw[0] += c1 - c0;
        double* hrow = Hs + 8 * b * 32;
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          bb[i] = __dsub_rn(bb[i], Ss[i * WS_SLD + lane]);
          x[i] = hrow[i * 32 + hoff[i & 3]];
        }
        double hv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < ((SKIP & 1) ? 0 : 8); ++i) {
          const double t = __dmul_rn(bb[i], gc[36 + i]);
          const double h = pos_part_ws(t);
          hv[i] = h;
#pragma unroll
          for (int l = i + 1; l < 8; ++l) bb[l] = fma(-gc[l * (l - 1) / 2 + i], h, bb[l]);
          hrow[i * 32 + hoff[i & 3]] = h;
          // G_kk((x-t)² - (h-t)²) = (x-h)(G_kk(x+h) - 2b_k), accumulated halved
          const double u = __dsub_rn(x[i], h), v = __dadd_rn(x[i], h);
          gain = fma(u, fma(gc[28 + i], v, -bb[i]), gain);
        }
        if (b + 1 < NB) nb_arrive(idH);
        if (PROF) pw[2] += clock64() - c1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (8 * b + i < rv) {
            hp[(long)(8 * b + i) * a.ld] = hv[i];
            const long long hb = __double_as_longlong(hv[i]);
            hmax = hb > hmax ? hb : hmax;
          }
        }
      }
      nf |= hmax >= 0x7FF0000000000000LL;
    }
  }
  if (!PERSIST) break;
  // ---- grid-wide end of sweep `sw`: stall rule on the total gain ----
  const long long tg0 = PROF ? clock64() : 0;
  {
    const double bg = block_reduce_sum_any(__dadd_rn(gain, gain), red);
    const int bnf = __syncthreads_or(nf);
    const unsigned target = (unsigned)(sw + 1) * gridDim.x;
    if (threadIdx.x == 0) {
      a.part[blockIdx.x] = bg;
      a.part_nf[blockIdx.x] = bnf;
      __threadfence();
      const unsigned prev = atomicAdd(&a.ctl->arrive, 1u);
      s_flag = prev == target - 1 ? 1 : 0;   // this CTA arrived last (used when sharded)
    }
    if (!a.dv) {
      // every CTA forms the same fixed-order total itself once all partials are in
      if (threadIdx.x == 0) {
        unsigned e;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(e) : "l"(&a.ctl->arrive) : "memory");
        } while (e < target);
      }
      __syncthreads();
      double v = 0.0;
      int f = 0;
      for (int b = threadIdx.x; b < (int)gridDim.x; b += 256) {
        v = __dadd_rn(v, __ldcg(a.part + b));
        f |= __ldcg(a.part_nf + b);
      }
      const double total = block_reduce_sum_any(v, red);
      f = __syncthreads_or(f);
      if (sw == 0) first_total = total;
      const bool stop = (sw + 1 >= a.max_sweeps) ||
                        (total <= __dmul_rn(a.stall, first_total < 0.0 ? 0.0 : first_total));
      if (blockIdx.x == 0 && threadIdx.x == 0) finish_sweep(a, total, f);   // bookkeeping (same rule)
      s_flag = stop ? 0 : 1;
    } else {
      // sharded: the last CTA exchanges the gain with the other ranks and publishes the decision
      __syncthreads();
      if (s_flag) {
        __threadfence();
        double v = 0.0;
        int f = 0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 256) {
          v = __dadd_rn(v, __ldcg(a.part + b));
          f |= __ldcg(a.part_nf + b);
        }
        double total = block_reduce_sum_any(v, red);
        f = __syncthreads_or(f);
        if (threadIdx.x == 0) {
          dist::allreduce_gain(*a.dv, total, f, &total, &f);
          finish_sweep(a, total, f);
          __threadfence();
          asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(&a.ctl->epoch), "r"((unsigned)(sw + 1))
                       : "memory");
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned e;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(e) : "l"(&a.ctl->epoch) : "memory");
        } while (e < (unsigned)(sw + 1));
        s_flag = *(volatile int*)&a.ctl->cont;
      }
    }
    __syncthreads();
    if (PROF) pw[3] += clock64() - tg0;
    if (!s_flag) break;
    gain = 0.0;
    nf = 0;
    src = a.H;
  }
  }
  if (PROF && lane == 0) {
    double* o = a.terms + ((long)blockIdx.x * 8 + warp) * 8;
    o[0] = (double)pw[0];
    o[1] = (double)pw[1];
    o[2] = (double)(clock64() - tk0);
    o[3] = (double)pw[2];
    o[4] = (double)pw[3];
  }
  if (!PERSIST) {
    const double bg = block_reduce_sum_any(__dadd_rn(gain, gain), red);
    nf = __syncthreads_or(nf);
    last_block_reduce_n<256>(a, bg, nf, red);
  }
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
  c->epoch = 0;
}

}  // namespace hals

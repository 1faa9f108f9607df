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
ENMF_DEV void last_block_reduce(const Args& a, double block_gain, int block_nf, double* red) {
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
  for (int b = threadIdx.x; b < (int)gridDim.x; b += NT) {
    v = __dadd_rn(v, __ldcg(a.part + b));
    nf |= __ldcg(a.part_nf + b);
  }
  const double total = block_reduce_sum<NT>(v, red);
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
  last_block_reduce(a, bg, nf, red);
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

// common.cuh — shared device-side definitions for the B200 enmf hot path.
//
// The whole translation unit is compiled with -fmad=false: every multiply-add
// that is meant to be fused is written as an explicit fma() (or a DMMA), so the
// elementwise and scalar code keeps the reference's separately-rounded
// arithmetic (matrix.hpp / engine.hpp) bit for bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/enmf_gpu.h"

#define ENMF_DEV __device__ __forceinline__

// Per-side control block of the multi-sweep HALS loop (nnls.hpp:154-176).
struct HalsCtl {
  double first_gain;     // gain of sweep 1
  double last_gain;      // gain of the most recent sweep
  int sweeps;            // sweeps performed in the current solve
  int cont;              // 1 while another sweep is due
  int nonfinite;         // last sweep wrote a non-finite value
  int degenerate;        // index+1 of a degenerate Gram diagonal (0 = none)
  unsigned arrive;       // block-arrival counter for the last-block reduction
  unsigned epoch;        // persistent sweep kernel: number of sweeps decided
};

// Device-resident run state: BetaSchedule (engine.hpp:63-70), err_prev, the
// iteration counter and every decision flag, so that a whole outer iteration
// runs as one CUDA graph with no host round trip.
struct DevState {
  double beta, beta_bar, beta_prev, gamma, gamma_bar, eta;  // BetaSchedule
  double beta_used;         // beta of the current iteration (0 if extrapolation off)
  double err_prev;
  double norm_x_sq, norm_x;
  double dot_hi, dot_lo;    // <W_n, X T^T> (double-double)
  double max_seconds;
  double last_elapsed;
  unsigned long long k;      // 1-based index of the iteration in flight
  unsigned long long max_iter;
  unsigned long long t0_ns;
  int active;               // 0 once stopped (error or wall budget)
  int error_code;           // ENMF_* of the failure that stopped the run
  int restarted;
  int reinit_events;        // bit0: W_y redrawn, bit1: target redrawn (this iteration)
  int reinit_flag[2];       // Gram diagonal check failed (0: W_y side, 1: T side)
  int extrapolation;
  int hp;
  int wall;
  int literal;
  int bpp_rounds[2];
  unsigned long long bpp_exchanges[2];
  unsigned arrive_dot;
  int pad;
  HalsCtl hals[2];          // 0: H update, 1: W update
};

ENMF_DEV bool dev_active(const DevState* st) { return *(volatile const int*)&st->active != 0; }

ENMF_DEV unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- error-free transformations / double-double ---------------------------
ENMF_DEV void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
ENMF_DEV void two_prod(double a, double b, double& p, double& e) {
  p = __dmul_rn(a, b);
  e = fma(a, b, -p);
}
// (hi, lo) += (bh, bl)
ENMF_DEV void dd_add(double& hi, double& lo, double bh, double bl) {
  double s, e;
  two_sum(hi, bh, s, e);
  e = __dadd_rn(e, __dadd_rn(lo, bl));
  hi = __dadd_rn(s, e);
  lo = __dsub_rn(e, __dsub_rn(hi, s));
}
// (hi, lo) += a*b exactly-rounded product accumulation
ENMF_DEV void dd_add_prod(double& hi, double& lo, double a, double b) {
  double p, pe;
  two_prod(a, b, p, pe);
  dd_add(hi, lo, p, pe);
}

// Neumaier CompensatedSum::add, linalg.hpp:29-37 (bitwise).
ENMF_DEV void neumaier_add(double& sum, double& c, double v) {
  const double t = __dadd_rn(sum, v);
  if (fabs(sum) >= fabs(v)) {
    c = __dadd_rn(c, __dadd_rn(__dsub_rn(sum, t), v));
  } else {
    c = __dadd_rn(c, __dadd_rn(__dsub_rn(v, t), sum));
  }
  sum = t;
}

// ---- std::mt19937_64 + rng.hpp helpers (device, single thread) ------------
struct DevMt64 {
  uint64_t mt[312];
  int idx;
};
ENMF_DEV void mt64_seed(DevMt64& g, uint64_t seed) {
  g.mt[0] = seed;
  for (int i = 1; i < 312; ++i) g.mt[i] = 6364136223846793005ULL * (g.mt[i - 1] ^ (g.mt[i - 1] >> 62)) + (uint64_t)i;
  g.idx = 312;
}
ENMF_DEV uint64_t mt64_next(DevMt64& g) {
  if (g.idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g.mt[i] & 0xFFFFFFFF80000000ULL) | (g.mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = g.mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g.mt[i] = v;
    }
    g.idx = 0;
  }
  uint64_t z = g.mt[g.idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}
// rng.hpp:30-49
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t mix_seed(uint64_t base, uint64_t a, uint64_t b) {
  const uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
  uint64_t h = mix64(base + kGolden);
  h = mix64(h ^ (a + kGolden));
  h = mix64(h ^ (b + kGolden));
  return h;
}
ENMF_DEV double uniform_unit(DevMt64& g) { return __dmul_rn((double)(mt64_next(g) >> 11), 0x1.0p-53); }

// ---- block reductions (deterministic: fixed tree) -------------------------
template <int NT>
ENMF_DEV void block_reduce_dd(double& hi, double& lo, double* sh_hi, double* sh_lo) {
  const int tid = threadIdx.x;
  sh_hi[tid] = hi;
  sh_lo[tid] = lo;
  __syncthreads();
#pragma unroll
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (tid < s) {
      double h = sh_hi[tid], l = sh_lo[tid];
      dd_add(h, l, sh_hi[tid + s], sh_lo[tid + s]);
      sh_hi[tid] = h;
      sh_lo[tid] = l;
    }
    __syncthreads();
  }
  hi = sh_hi[0];
  lo = sh_lo[0];
  __syncthreads();
}

template <int NT>
ENMF_DEV double block_reduce_sum(double v, double* sh) {
  const int tid = threadIdx.x;
  sh[tid] = v;
  __syncthreads();
#pragma unroll
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (tid < s) sh[tid] = __dadd_rn(sh[tid], sh[tid + s]);
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// Any block size (multiple of 32): xor-butterfly inside each warp, then warp
// partials summed in warp order by thread 0.  Deterministic; result broadcast.
ENMF_DEV double block_reduce_sum_any(double v, double* sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) sh[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = sh[0];
    for (int w = 1; w < nw; ++w) s = __dadd_rn(s, sh[w]);
    sh[32] = s;
  }
  __syncthreads();
  const double r = sh[32];
  __syncthreads();
  return r;
}

// D(8×8) += A(8×4) · B(4×8) in FP64 on the tensor pipe (one DMMA.8x8x4 on sm_100a).
ENMF_DEV void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NT>
ENMF_DEV int block_reduce_or(int v, int* sh) {
  const int r = __syncthreads_or(v);
  (void)sh;
  return r;
}

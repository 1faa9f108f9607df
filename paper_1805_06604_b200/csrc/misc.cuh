// misc.cuh — elementwise, reduction and decision kernels of step()/run().
//
//   run_begin / iter_begin      run loop bookkeeping, wall budget (engine.hpp:461-466,505-506)
//   reinit_fixup                gram_with_reinit + reinit_columns (engine.hpp:268-296)
//   extrap                      extrapolate + clamp_nonnegative (engine.hpp:102-113, matrix.hpp:114-116)
//   finalize                    W/H extrapolation + restart/accept (engine.hpp:386-397, 420-429)
//   frob_partial/frob_final     frob_norm_sq (linalg.hpp:160-171), double-double
//   dot_partial                 <W_n, X Tᵀ> of fast_error (engine.hpp:129-130), double-double
//   decide                      fast_error tail + NaN guard + restart test + update_beta
//                               + IterationRecord (engine.hpp:131-136, 413-439, 88-99)
//   *_exact                     the reference's sequential Neumaier order (debug/parity mode)
#pragma once

#include "common.cuh"

namespace misc {

constexpr int NT = 256;

__global__ void run_begin(DevState* st) { st->t0_ns = globaltimer_ns(); }

ENMF_DEV double elapsed_s(const DevState* st) {
  return (double)(globaltimer_ns() - st->t0_ns) * 1e-9;
}

// Start of outer iteration k (engine.hpp:505-507, 315).
__global__ void iter_begin(DevState* st) {
  if (!st->active) return;
  if (st->wall && elapsed_s(st) >= st->max_seconds) {  // budget exhausted: stop, no record
    st->active = 0;
    return;
  }
  st->k += 1;
  st->beta_used = st->extrapolation ? st->beta : 0.0;
  st->reinit_events = 0;
  st->reinit_flag[0] = st->reinit_flag[1] = 0;
}

// gram_with_reinit (engine.hpp:279-296) for the factor whose columns are the
// rows of A (r rows, K contiguous values each).  G already holds gram(A);
// if a diagonal is !(> 1e-16 max diag) the offending rows are redrawn from
// mt19937_64(mix_seed(reinit_seed, salt, attempt)) in ascending order, each
// filled first to last, and the Gram is recomputed (reference order).
__global__ void __launch_bounds__(NT) reinit_fixup(double* A, long lda, int r, int K, double* G,
                                                   uint64_t reinit_seed, int side, DevState* st) {
  if (!dev_active(st)) return;
  __shared__ int bad[1024];
  __shared__ int nbad;
  const uint64_t salt = 2ULL * st->k + (uint64_t)side;
  for (uint64_t attempt = 0;; ++attempt) {
    if (threadIdx.x == 0) {
      double maxd = 0.0;
      for (int i = 0; i < r; ++i) maxd = (maxd < G[i * r + i]) ? G[i * r + i] : maxd;
      const double fl = __dmul_rn(1e-16, maxd);
      int nb = 0;
      for (int kk = 0; kk < r; ++kk)
        if (!(G[kk * r + kk] > fl) && nb < 1024) bad[nb++] = kk;
      nbad = nb;
    }
    __syncthreads();
    if (nbad == 0) return;
    if (attempt > (uint64_t)r + 2) {
      if (threadIdx.x == 0) {
        st->error_code = ENMF_NO_CONVERGENCE;
        st->active = 0;
      }
      return;
    }
    if (threadIdx.x == 0) {
      DevMt64 gen;
      mt64_seed(gen, mix_seed(reinit_seed, salt, attempt));
      for (int q = 0; q < nbad; ++q) {
        double* row = A + (long)bad[q] * lda;
        for (int i = 0; i < K; ++i) row[i] = uniform_unit(gen);
      }
      st->reinit_events |= 1 << side;
      __threadfence_block();
    }
    __syncthreads();
    for (int e = threadIdx.x; e < r * r; e += NT) {
      const int kk = e / r, j = e % r;
      if (kk > j) continue;
      const double* ak = A + (long)kk * lda;
      const double* aj = A + (long)j * lda;
      double s = 0.0;
      for (int i = 0; i < K; ++i) s = __dadd_rn(s, __dmul_rn(ak[i], aj[i]));
      G[kk * r + j] = s;
      G[j * r + kk] = s;
    }
    __syncthreads();
  }
}

// out = next + beta*(next - prev) (+ clamp), beta from the run state.
__global__ void extrap(const double* __restrict__ next, const double* __restrict__ prev, double* __restrict__ out,
                       long count, int clamp, const DevState* st) {
  if (!dev_active(st)) return;
  const double beta = st->beta_used;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x) {
    const double nv = next[i];
    double v = __dadd_rn(nv, __dmul_rn(beta, __dsub_rn(nv, prev[i])));
    if (clamp) v = v > 0.0 ? v : 0.0;
    out[i] = v;
  }
}

__global__ void copy(const double* __restrict__ src, double* __restrict__ dst, long count, const DevState* st) {
  if (st && !dev_active(st)) return;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// End of iteration: W extrapolation (always after the W update), the late H
// extrapolation for hp = 1, and the restart/accept copies.
//   mode_h: 0 = hp>=2 (H_y already set), 1 = hp==1 (compute H_y), 2 = literal hp1 (H_y set)
__global__ void finalize(double* __restrict__ WT, double* __restrict__ WyT, const double* __restrict__ WnT, long wcount,
                         double* __restrict__ H, double* __restrict__ Hy, const double* __restrict__ Hn, long hcount,
                         int mode_h, const DevState* st) {
  if (!dev_active(st)) return;
  const bool restart = st->restarted != 0;
  const bool ex = st->extrapolation != 0;
  const double beta = st->beta_used;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < wcount; i += stride) {
    const double wn = WnT[i];
    if (restart) {
      WyT[i] = WT[i];
    } else {
      WyT[i] = ex ? __dadd_rn(wn, __dmul_rn(beta, __dsub_rn(wn, WT[i]))) : wn;
      WT[i] = wn;
    }
  }
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < hcount; i += stride) {
    const double hn = Hn[i];
    if (restart) {
      Hy[i] = H[i];
    } else {
      if (mode_h == 1) Hy[i] = ex ? __dadd_rn(hn, __dmul_rn(beta, __dsub_rn(hn, H[i]))) : hn;
      H[i] = hn;
    }
  }
}

// ---- reductions ------------------------------------------------------------
// Per-block double-double partial sums of x[i]^2 (frob) or a[i]*b[i] (dot).
__global__ void __launch_bounds__(NT) dd_partial(const double* __restrict__ a, const double* __restrict__ b, long count,
                                                 double* part_hi, double* part_lo, const DevState* st) {
  if (st && !dev_active(st)) return;
  __shared__ double sh[NT], sl[NT];
  double hi = 0.0, lo = 0.0;
  for (long i = blockIdx.x * (long)NT + threadIdx.x; i < count; i += (long)gridDim.x * NT) {
    const double x = a[i];
    dd_add_prod(hi, lo, x, b ? b[i] : x);
  }
  block_reduce_dd<NT>(hi, lo, sh, sl);
  if (threadIdx.x == 0) {
    part_hi[blockIdx.x] = hi;
    part_lo[blockIdx.x] = lo;
  }
}

// Fixed-order combination of the partials; writes (hi, lo) to out[0..1].
__global__ void __launch_bounds__(NT) dd_final(const double* part_hi, const double* part_lo, int nparts, double* out,
                                               const DevState* st) {
  if (st && !dev_active(st)) return;
  __shared__ double sh[NT], sl[NT];
  double hi = 0.0, lo = 0.0;
  for (int i = threadIdx.x; i < nparts; i += NT) dd_add(hi, lo, part_hi[i], part_lo[i]);
  block_reduce_dd<NT>(hi, lo, sh, sl);
  if (threadIdx.x == 0) {
    out[0] = hi;
    out[1] = lo;
  }
}

// optimal_beta_linesearch (engine.hpp:522-540) terms.  Element (i,j) of DH = (W_n − W)·H_y
// and WH = W_n·H_y is formed exactly as the reference's multiply forms it (linalg.hpp:174-189:
// diff rounded first, products added in ascending p from 0.0, no contraction), then
// accumulated in double-double: q=0 Σ DH², q=1 Σ WH·DH, q=2 Σ X·DH (dense X only).
// Element e = i·n + j with j fastest, so H_y rows are read coalesced.  part: 6 per block.
__global__ void __launch_bounds__(NT) linesearch_terms(const double* __restrict__ x, const double* __restrict__ wn,
                                                       const double* __restrict__ w, const double* __restrict__ h,
                                                       long m, long n, int r, double* __restrict__ part) {
  __shared__ double sh[NT], sl[NT];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (long e = blockIdx.x * (long)NT + threadIdx.x; e < m * n; e += (long)gridDim.x * NT) {
    const long i = e / n, j = e - i * n;
    const double* a = wn + i * r;
    const double* b = w + i * r;
    double dh = 0.0, wh = 0.0;
    for (int p = 0; p < r; ++p) {
      const double hp = h[(long)p * n + j];
      dh = __dadd_rn(dh, __dmul_rn(__dsub_rn(a[p], b[p]), hp));
      wh = __dadd_rn(wh, __dmul_rn(a[p], hp));
    }
    dd_add_prod(acc[0], acc[1], dh, dh);
    dd_add_prod(acc[2], acc[3], wh, dh);
    if (x) dd_add_prod(acc[4], acc[5], x[e], dh);
  }
  for (int q = 0; q < 3; ++q) {
    double hi = acc[2 * q], lo = acc[2 * q + 1];
    block_reduce_dd<NT>(hi, lo, sh, sl);
    if (threadIdx.x == 0) {
      part[6 * blockIdx.x + 2 * q] = hi;
      part[6 * blockIdx.x + 2 * q + 1] = lo;
    }
    __syncthreads();
  }
}

// Σ X·DH over the stored entries of a CSR X (frob_inner(SparseMatrix, DenseMatrix),
// linalg.hpp:192-205), one thread per row; part[2·block .. +1] = (hi, lo).
__global__ void __launch_bounds__(NT) linesearch_xdh_csr(const unsigned long long* __restrict__ off,
                                                         const unsigned long long* __restrict__ idx,
                                                         const double* __restrict__ val, const double* __restrict__ wn,
                                                         const double* __restrict__ w, const double* __restrict__ h,
                                                         long m, long n, int r, double* __restrict__ part) {
  __shared__ double sh[NT], sl[NT];
  double hi = 0.0, lo = 0.0;
  for (long i = blockIdx.x * (long)NT + threadIdx.x; i < m; i += (long)gridDim.x * NT) {
    const double* a = wn + i * r;
    const double* b = w + i * r;
    for (unsigned long long q = off[i]; q < off[i + 1]; ++q) {
      const long j = (long)idx[q];
      double dh = 0.0;
      for (int p = 0; p < r; ++p) dh = __dadd_rn(dh, __dmul_rn(__dsub_rn(a[p], b[p]), h[(long)p * n + j]));
      dd_add_prod(hi, lo, val[q], dh);
    }
  }
  block_reduce_dd<NT>(hi, lo, sh, sl);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = hi;
    part[2 * blockIdx.x + 1] = lo;
  }
}

// Fixed-order combination of `streams` interleaved (hi, lo) partial streams:
// part[(b·streams + q)·2 + {0,1}] → out[2q], out[2q+1].  One block.
__global__ void __launch_bounds__(NT) dd_final_multi(const double* part, int nparts, int streams, double* out) {
  __shared__ double sh[NT], sl[NT];
  for (int q = 0; q < streams; ++q) {
    double hi = 0.0, lo = 0.0;
    for (int b = threadIdx.x; b < nparts; b += NT) dd_add(hi, lo, part[(b * streams + q) * 2], part[(b * streams + q) * 2 + 1]);
    block_reduce_dd<NT>(hi, lo, sh, sl);
    if (threadIdx.x == 0) {
      out[2 * q] = hi;
      out[2 * q + 1] = lo;
    }
    __syncthreads();
  }
}

// Reference-order Neumaier sum of x[i]^2 or a[i]*b[i] (frob_norm_sq, frob_inner), one thread.
// For the fast_error cross term: a = W_nᵀ (r×m), b = P (r×m) visited in W_n's
// row-major order (i outer, k inner), term = -2*w*x.
__global__ void neumaier_exact(const double* a, const double* b, long count, int mode, int r, long m, double* out,
                               const DevState* st) {
  if (st && !dev_active(st)) return;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0, c = 0.0;
  if (mode == 1 && st) neumaier_add(s, c, st->norm_x_sq);  // acc.add(norm_x_sq), engine.hpp:127
  if (mode == 0) {
    for (long i = 0; i < count; ++i) neumaier_add(s, c, __dmul_rn(a[i], a[i]));
  } else {
    for (long i = 0; i < m; ++i)
      for (int k = 0; k < r; ++k) {
        const long e = (long)k * m + i;
        neumaier_add(s, c, __dmul_rn(__dmul_rn(-2.0, a[e]), b[e]));
      }
  }
  out[0] = s;
  out[1] = c;
}

// fast_error tail + decisions.  dd_dot: (hi, lo) of <W_n, XTᵀ> (fast) or the
// Neumaier (sum, c) of the -2<W_n, XTᵀ> terms (exact).  gwn = gram(W_n), gw = T Tᵀ.
// k == 0 records the initial pair (engine.hpp:487-503).
__global__ void __launch_bounds__(NT) decide(DevState* st, const double* dd_dot, const double* gwn, const double* gw,
                                             int r, int exact, enmf_gpu_iter* recs, unsigned long long init) {
  if (!dev_active(st)) return;
  __shared__ double sh[NT], sl[NT];
  double err;
  if (exact) {
    if (threadIdx.x != 0) return;
    // CompensatedSum: add(norm_x_sq), then the -2 w x terms (already accumulated
    // in order as (sum, c) starting from norm_x_sq? no: restart from scratch)
    // The exact path accumulates everything in one Neumaier stream below.
    double s = dd_dot[0], c = dd_dot[1];  // stream already seeded with norm_x_sq
    for (int i = 0; i < r * r; ++i) neumaier_add(s, c, __dmul_rn(gwn[i], gw[i]));
    const double v = __dadd_rn(s, c);
    err = __dsqrt_rn(0.0 < v ? v : 0.0);
  } else {
    double hi = 0.0, lo = 0.0;
    for (int i = threadIdx.x; i < r * r; i += NT) dd_add_prod(hi, lo, gwn[i], gw[i]);
    block_reduce_dd<NT>(hi, lo, sh, sl);
    if (threadIdx.x != 0) return;
    // ||X||^2 - 2<W,XHᵀ> + <WᵀW,HHᵀ> in double-double
    double sh_ = st->norm_x_sq, sl_ = 0.0;
    dd_add(sh_, sl_, __dmul_rn(-2.0, dd_dot[0]), __dmul_rn(-2.0, dd_dot[1]));
    dd_add(sh_, sl_, hi, lo);
    const double v = __dadd_rn(sh_, sl_);
    err = __dsqrt_rn(0.0 < v ? v : 0.0);
  }
  const unsigned long long k = init ? 0ULL : st->k;
  enmf_gpu_iter rec;
  rec.iteration = k;
  rec.elapsed_seconds = 0.0;
  rec.error = err;
  rec.relative_error = st->norm_x > 0.0 ? __ddiv_rn(err, st->norm_x) : 0.0;
  rec.beta = init ? (st->extrapolation ? st->beta : 0.0) : st->beta_used;
  rec.restarted = 0;
  rec.inner_h_count = 0;
  rec.inner_w_count = 0;
  rec.reinit_events = 0;
  if (init) {
    st->err_prev = err;
    st->restarted = 0;
  } else {
    if (!isfinite(err)) {  // engine.hpp:413-416
      st->error_code = ENMF_NON_FINITE;
      st->active = 0;
      return;
    }
    const bool restart = err > st->err_prev;
    st->restarted = restart ? 1 : 0;
    if (st->extrapolation) {  // update_beta, engine.hpp:88-99
      const bool dec = err <= st->err_prev;
      const double used = st->beta;
      if (dec) {
        const double gb = __dmul_rn(st->gamma, st->beta);
        st->beta = gb < st->beta_bar ? gb : st->beta_bar;
        const double gbb = __dmul_rn(st->gamma_bar, st->beta_bar);
        st->beta_bar = gbb < 1.0 ? gbb : 1.0;
      } else {
        st->beta = __ddiv_rn(st->beta, st->eta);
        st->beta_bar = st->beta_prev;
      }
      st->beta_prev = used;
    }
    st->err_prev = err;
    rec.restarted = restart ? 1 : 0;
    rec.inner_h_count = st->hals[0].sweeps ? st->hals[0].sweeps : st->bpp_rounds[0];
    rec.inner_w_count = st->hals[1].sweeps ? st->hals[1].sweeps : st->bpp_rounds[1];
    rec.reinit_events = st->reinit_events;
  }
  if (st->wall) {
    double el = elapsed_s(st);
    if (!init && el <= st->last_elapsed) el = nextafter(st->last_elapsed, __longlong_as_double(0x7ff0000000000000LL));
    st->last_elapsed = el;
    rec.elapsed_seconds = el;
  }
  recs[k] = rec;
}

// ||X||^2 from a (hi, lo) / (sum, c) pair.
__global__ void set_norm(DevState* st, const double* dd) {
  if (!dev_active(st)) return;
  const double v = __dadd_rn(dd[0], dd[1]);
  st->norm_x_sq = v;
  st->norm_x = __dsqrt_rn(v);
}

// fast_error tail without run state (standalone kernel API).
__global__ void __launch_bounds__(NT) fast_error_tail(double nx2, const double* dd_dot, const double* gwn,
                                                       const double* hht, int r, int exact, double* out) {
  __shared__ double sh[NT], sl[NT];
  if (exact) {
    if (threadIdx.x != 0) return;
    double s = dd_dot[0], c = dd_dot[1];
    for (int i = 0; i < r * r; ++i) neumaier_add(s, c, __dmul_rn(gwn[i], hht[i]));
    const double v = __dadd_rn(s, c);
    *out = __dsqrt_rn(0.0 < v ? v : 0.0);
    return;
  }
  double hi = 0.0, lo = 0.0;
  for (int i = threadIdx.x; i < r * r; i += NT) dd_add_prod(hi, lo, gwn[i], hht[i]);
  block_reduce_dd<NT>(hi, lo, sh, sl);
  if (threadIdx.x != 0) return;
  double a = nx2, b = 0.0;
  dd_add(a, b, __dmul_rn(-2.0, dd_dot[0]), __dmul_rn(-2.0, dd_dot[1]));
  dd_add(a, b, hi, lo);
  const double v = __dadd_rn(a, b);
  *out = __dsqrt_rn(0.0 < v ? v : 0.0);
}

// Tiled transpose: out (cols×rows) = in (rows×cols)ᵀ.
__global__ void transpose(const double* __restrict__ in, double* __restrict__ out, int rows, int cols) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = by + j, c = bx + threadIdx.x;
    if (r < rows && c < cols) tile[j][threadIdx.x] = in[(long)r * cols + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int c = bx + j, r = by + threadIdx.x;
    if (r < rows && c < cols) out[(long)c * rows + r] = tile[threadIdx.x][j];
  }
}

// Input validation on device-resident factors: finite and nonnegative (engine.hpp:457-459).
// nonneg = 0: finiteness only (the DenseMatrix invariant for X, matrix.hpp:43-51).
__global__ void check_factor(const double* a, long count, int* bad, int nonneg) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x) {
    const double v = a[i];
    if (!isfinite(v) || (nonneg && !(v >= 0.0))) atomicOr(bad, 1);
  }
}

}  // namespace misc

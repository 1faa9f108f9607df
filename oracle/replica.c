/*
 * replica.c — bit-exact MULTI-THREADED restatement of the reference's dense
 * hot path ("for C5 ... a bit-exact multi-threaded replica").
 *
 * TEST INFRASTRUCTURE ONLY (linked into oracle/liboracle.so; used by tests/,
 * tests/golden/make_golden_c5.py and bench.py's --impl reference / cpu_baseline
 * legs).  The product never calls it.
 *
 * Every output element keeps the reference's sequential summation order and
 * separately rounded multiply/add (built with -ffp-contract=off, no fast-math),
 * so the results are bitwise identical to the single-threaded reference; only
 * the ORDER IN WHICH INDEPENDENT ELEMENTS ARE PRODUCED changes:
 *   cross_wx  (linalg.hpp:67-83)   out(k,j) = Σ_i w(i,k)·x(i,j), i ascending:
 *             threads over column blocks of j, i innermost in registers.
 *   cross_xht (linalg.hpp:107-124) out(i,k) = Σ_j x(i,j)·h(k,j), j ascending:
 *             threads over row blocks of i, j chunks with the partial sums
 *             stored and reloaded between chunks (order unchanged).
 *   gram      (linalg.hpp:49-64)   g(k,j) = Σ_i a(i,k)·a(i,j), i ascending:
 *             threads over k.
 *   hals_solve (nnls.hpp:111-176): within a sweep the columns t are independent
 *             (row k of column t reads rows j of the same column only), so
 *             threads own column blocks for the whole sweep; the per-row gain
 *             terms d_old² − d_new² are stored and summed sequentially in t per
 *             row, then the row gains are added in k order — the reference's
 *             exact gain, hence the same stall decisions.
 * Pinned bitwise against oracle/_ref (the reference compiled in place) in
 * tests/test_oracle.py::test_replica_bitwise_vs_reference.
 *
 * Also: the tiled C5 data generator (orc_gen_tiled), deterministic for any
 * thread count.
 */
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#include "enmf_oracle.h"

typedef double v4d __attribute__((vector_size(32)));

static inline v4d v_load(const double* p) { v4d v; memcpy(&v, p, sizeof v); return v; }
static inline void v_store(double* p, v4d v) { memcpy(p, &v, sizeof v); }
static inline v4d v_bcast(double s) { return (v4d){s, s, s, s}; }

int g_orc_threads = 1;

void orc_set_threads(int n) { g_orc_threads = n < 1 ? 1 : n; }
int orc_get_threads(void) { return g_orc_threads; }

/* ------------------------------------------------------------- cross_wx */
/* out (r×n) = wᵀx, linalg.hpp:67-83.  Per element the sum runs over i ascending from 0.0. */
void rep_cross_wx(const double* w, const double* x, size_t m, size_t n, size_t r, double* out) {
  /* the x rows of a chunk sit n·8 bytes apart — the same L1 sets for every row — so each
   * (row chunk, column block) is first copied into a contiguous per-thread buffer */
  enum { JB = 64, IC = 64 };
  const size_t nblk = (n + JB - 1) / JB;
  memset(out, 0, sizeof(double) * r * n);
#pragma omp parallel num_threads(g_orc_threads)
  {
    double* xb = (double*)aligned_alloc(64, sizeof(double) * IC * JB);
#pragma omp for schedule(dynamic, 1)
    for (size_t b = 0; b < nblk; ++b) {
      const size_t j0 = b * JB, j1 = j0 + JB < n ? j0 + JB : n, jw = j1 - j0;
      for (size_t i0 = 0; i0 < m; i0 += IC) {
        const size_t i1 = i0 + IC < m ? i0 + IC : m;
        for (size_t i = i0; i < i1; ++i) memcpy(xb + (i - i0) * JB, x + i * n + j0, sizeof(double) * jw);
        size_t k = 0;
        for (; k + 4 <= r; k += 4) {
          size_t j = 0;
          for (; j + 8 <= jw; j += 8) {
            double* o = out + j0 + j;
            v4d a00 = v_load(o + (k + 0) * n), a01 = v_load(o + (k + 0) * n + 4);
            v4d a10 = v_load(o + (k + 1) * n), a11 = v_load(o + (k + 1) * n + 4);
            v4d a20 = v_load(o + (k + 2) * n), a21 = v_load(o + (k + 2) * n + 4);
            v4d a30 = v_load(o + (k + 3) * n), a31 = v_load(o + (k + 3) * n + 4);
            for (size_t i = i0; i < i1; ++i) {
              const double* xi = xb + (i - i0) * JB + j;
              const double* wi = w + i * r + k;
              const v4d x0 = v_load(xi), x1 = v_load(xi + 4);
              v4d s;
              s = v_bcast(wi[0]); a00 = a00 + s * x0; a01 = a01 + s * x1;
              s = v_bcast(wi[1]); a10 = a10 + s * x0; a11 = a11 + s * x1;
              s = v_bcast(wi[2]); a20 = a20 + s * x0; a21 = a21 + s * x1;
              s = v_bcast(wi[3]); a30 = a30 + s * x0; a31 = a31 + s * x1;
            }
            v_store(o + (k + 0) * n, a00); v_store(o + (k + 0) * n + 4, a01);
            v_store(o + (k + 1) * n, a10); v_store(o + (k + 1) * n + 4, a11);
            v_store(o + (k + 2) * n, a20); v_store(o + (k + 2) * n + 4, a21);
            v_store(o + (k + 3) * n, a30); v_store(o + (k + 3) * n + 4, a31);
          }
          for (; j < jw; ++j)
            for (size_t kk = k; kk < k + 4; ++kk) {
              double a = out[kk * n + j0 + j];
              for (size_t i = i0; i < i1; ++i) a += w[i * r + kk] * xb[(i - i0) * JB + j];
              out[kk * n + j0 + j] = a;
            }
        }
        for (; k < r; ++k)
          for (size_t j = 0; j < jw; ++j) {
            double a = out[k * n + j0 + j];
            for (size_t i = i0; i < i1; ++i) a += w[i * r + k] * xb[(i - i0) * JB + j];
            out[k * n + j0 + j] = a;
          }
      }
    }
    free(xb);
  }
}

/* ------------------------------------------------------------ cross_xht */
/* out (m×r) = x·hᵀ, linalg.hpp:107-124.  Per element the sum runs over j ascending from 0.0. */
void rep_cross_xht(const double* x, const double* h, size_t m, size_t n, size_t r, double* out) {
  const size_t IB = 64, JC = 512;
  double* ht = (double*)malloc(sizeof(double) * n * r);   /* hᵀ, n×r (exact copy) */
#pragma omp parallel for schedule(static) num_threads(g_orc_threads)
  for (size_t j = 0; j < n; ++j)
    for (size_t k = 0; k < r; ++k) ht[j * r + k] = h[k * n + j];
  memset(out, 0, sizeof(double) * m * r);
  const size_t nblk = (m + IB - 1) / IB;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_orc_threads)
  for (size_t b = 0; b < nblk; ++b) {
    const size_t i0 = b * IB, i1 = i0 + IB < m ? i0 + IB : m;
    for (size_t jc = 0; jc < n; jc += JC) {
      const size_t je = jc + JC < n ? jc + JC : n;
      size_t k = 0;
      for (; k + 8 <= r; k += 8) {
        size_t i = i0;
        for (; i + 4 <= i1; i += 4) {
          double* o0 = out + (i + 0) * r + k;
          double* o1 = out + (i + 1) * r + k;
          double* o2 = out + (i + 2) * r + k;
          double* o3 = out + (i + 3) * r + k;
          v4d a00 = v_load(o0), a01 = v_load(o0 + 4), a10 = v_load(o1), a11 = v_load(o1 + 4);
          v4d a20 = v_load(o2), a21 = v_load(o2 + 4), a30 = v_load(o3), a31 = v_load(o3 + 4);
          const double* x0 = x + (i + 0) * n;
          const double* x1 = x + (i + 1) * n;
          const double* x2 = x + (i + 2) * n;
          const double* x3 = x + (i + 3) * n;
          for (size_t j = jc; j < je; ++j) {
            const double* hj = ht + j * r + k;
            const v4d h0 = v_load(hj), h1 = v_load(hj + 4);
            v4d s;
            s = v_bcast(x0[j]); a00 = a00 + s * h0; a01 = a01 + s * h1;
            s = v_bcast(x1[j]); a10 = a10 + s * h0; a11 = a11 + s * h1;
            s = v_bcast(x2[j]); a20 = a20 + s * h0; a21 = a21 + s * h1;
            s = v_bcast(x3[j]); a30 = a30 + s * h0; a31 = a31 + s * h1;
          }
          v_store(o0, a00); v_store(o0 + 4, a01); v_store(o1, a10); v_store(o1 + 4, a11);
          v_store(o2, a20); v_store(o2 + 4, a21); v_store(o3, a30); v_store(o3 + 4, a31);
        }
        for (; i < i1; ++i)
          for (size_t kk = k; kk < k + 8; ++kk) {
            double a = out[i * r + kk];
            for (size_t j = jc; j < je; ++j) a += x[i * n + j] * ht[j * r + kk];
            out[i * r + kk] = a;
          }
      }
      for (; k < r; ++k)
        for (size_t i = i0; i < i1; ++i) {
          double a = out[i * r + k];
          for (size_t j = jc; j < je; ++j) a += x[i * n + j] * ht[j * r + k];
          out[i * r + k] = a;
        }
    }
  }
  free(ht);
}

/* ----------------------------------------------------------------- gram */
/* g (r×r) = aᵀa for a (rows×r) row-major, linalg.hpp:49-64: upper triangle over i ascending,
 * then mirrored. */
void rep_gram(const double* a, size_t rows, size_t r, double* g) {
  memset(g, 0, sizeof(double) * r * r);
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_orc_threads)
  for (size_t k = 0; k < r; ++k) {
    double* gk = g + k * r;
    size_t j = k;
    for (; j + 16 <= r; j += 16) {
      v4d a0 = v_bcast(0.0), a1 = a0, a2 = a0, a3 = a0;
      for (size_t i = 0; i < rows; ++i) {
        const double* ai = a + i * r;
        const v4d s = v_bcast(ai[k]);
        a0 = a0 + s * v_load(ai + j);
        a1 = a1 + s * v_load(ai + j + 4);
        a2 = a2 + s * v_load(ai + j + 8);
        a3 = a3 + s * v_load(ai + j + 12);
      }
      v_store(gk + j, a0); v_store(gk + j + 4, a1); v_store(gk + j + 8, a2); v_store(gk + j + 12, a3);
    }
    for (; j < r; ++j) {
      double s = 0.0;
      for (size_t i = 0; i < rows; ++i) s += a[i * r + k] * a[i * r + j];
      gk[j] = s;
    }
  }
  for (size_t k = 0; k < r; ++k)
    for (size_t j = k + 1; j < r; ++j) g[j * r + k] = g[k * r + j];
}

/* gram of the columns of t (r×n): gram(tᵀ), the rows of tᵀ in order. */
void rep_gram_rows(const double* t, size_t r, size_t n, double* g) {
  double* tt = (double*)malloc(sizeof(double) * n * r);
#pragma omp parallel for schedule(static) num_threads(g_orc_threads)
  for (size_t i = 0; i < n; ++i)
    for (size_t k = 0; k < r; ++k) tt[i * r + k] = t[k * n + i];
  rep_gram(tt, n, r, g);
  free(tt);
}

/* ----------------------------------------------------------- hals_solve */
/* nnls.hpp:154-176 with hals_row_update_impl (:111-136).  h is r×n row-major. */
int rep_hals_solve(const double* gram, const double* cross, const double* h0, size_t r, size_t n,
                   uint64_t max_sweeps, double stall_fraction, double* h, int32_t* sweeps) {
  double maxd = 0.0;                                        /* nnls.hpp:99-103 */
  for (size_t i = 0; i < r; ++i) maxd = (maxd < gram[i * r + i]) ? gram[i * r + i] : maxd;
  const double floor_ = 1e-16 * maxd;
  for (size_t k = 0; k < r; ++k)
    if (!(gram[k * r + k] > floor_)) {   /* the reference throws DegenerateColumn at row k */
      if (sweeps) *sweeps = 1;
      return ENMF_DEGENERATE_COLUMN;
    }
  if (h != h0) memcpy(h, h0, sizeof(double) * r * n);
  double* term = (double*)malloc(sizeof(double) * r * n);
  /* (the local column-block copy holds r <= 128 rows; larger r sweeps h in place) */
  double* rowg = (double*)malloc(sizeof(double) * r);
  const size_t CB = 32;
  const size_t nblk = (n + CB - 1) / CB;
  double first_gain = 0.0;
  uint64_t sweep;
  for (sweep = 1;; ++sweep) {
#pragma omp parallel num_threads(g_orc_threads)
    {
      /* the column block's rows of h sit n·8 bytes apart (the same L1 sets): the sweep runs on a
       * contiguous copy hb[j][0..CB) and writes it back */
      double hb[128 * 32];
      double s[32];
#pragma omp for schedule(dynamic, 1)
      for (size_t b = 0; b < nblk; ++b) {
        const size_t t0 = b * CB, t1 = t0 + CB < n ? t0 + CB : n, tw = t1 - t0;
        const int local = r <= 128;
        if (local)
          for (size_t j = 0; j < r; ++j) memcpy(hb + j * CB, h + j * n + t0, sizeof(double) * tw);
        for (size_t k = 0; k < r; ++k) {
          const double gkk = gram[k * r + k];
          const double* ck = cross + k * n + t0;
          const double* hbase = local ? hb : h + t0;
          const size_t hs = local ? CB : n;
          size_t t = 0;
          if (tw == 32) {
            v4d a[8];
            for (int u = 0; u < 8; ++u) a[u] = v_load(ck + 4 * u);
            for (size_t j = 0; j < r; ++j) {
              if (j == k) continue;
              const double gkj = gram[k * r + j];
              if (gkj == 0.0) continue;
              const double* hj = hbase + j * hs;
              const v4d g = v_bcast(gkj);
              for (int u = 0; u < 8; ++u) a[u] = a[u] - g * v_load(hj + 4 * u);
            }
            for (int u = 0; u < 8; ++u) v_store(s + 4 * u, a[u]);
            t = 32;
          }
          for (; t < tw; ++t) {
            double a = ck[t];
            for (size_t j = 0; j < r; ++j) {
              if (j == k) continue;
              const double gkj = gram[k * r + j];
              if (gkj == 0.0) continue;
              a -= gkj * hbase[j * hs + t];
            }
            s[t] = a;
          }
          double* hk = (double*)hbase + k * hs;
          double* tk = term + k * n + t0;
          for (t = 0; t < tw; ++t) {
            const double target = s[t] / gkk;
            const double next = target > 0.0 ? target : 0.0;
            const double d_old = hk[t] - target;
            const double d_new = next - target;
            tk[t] = d_old * d_old - d_new * d_new;
            hk[t] = next;
          }
        }
        if (local)
          for (size_t j = 0; j < r; ++j) memcpy(h + j * n + t0, hb + j * CB, sizeof(double) * tw);
      }
    }
#pragma omp parallel for schedule(static) num_threads(g_orc_threads)
    for (size_t k = 0; k < r; ++k) {
      const double* tk = term + k * n;
      double g = 0.0;
      for (size_t t = 0; t < n; ++t) g += tk[t];
      rowg[k] = gram[k * r + k] * g;
    }
    double gain = 0.0;
    for (size_t k = 0; k < r; ++k) gain += rowg[k];
    if (sweep == 1) first_gain = gain;
    if (sweep >= max_sweeps) break;
    if (gain <= stall_fraction * (first_gain < 0.0 ? 0.0 : first_gain)) break;
  }
  free(term);
  free(rowg);
  if (sweeps) *sweeps = (int32_t)sweep;
  return ENMF_OK;
}

/* ------------------------------------------------------ tiled generator */
/* BASELINE configs[4] (C5) data on T×T tiles, each from its own mt19937_64 stream, so the
 * matrix is identical for any thread count and any rank can build any block of it:
 *   W0 row block bi:    uniform[0,1), row-major, stream mix_seed(seed, 1, bi);
 *   H0 column block bj: uniform[0,1), for k: for j in block, stream mix_seed(seed, 2, bj);
 *   X tile (bi,bj):     Σ_k W0(i,k)·H0(k,j) (k ascending from 0.0, data.hpp:76-80's multiply
 *                       order) + 0.01·|N(0,1)|, one Box–Muller normal per entry, row-major in
 *                       the tile, stream mix_seed(seed, 3, bi·nbj + bj).
 * which = 5 only (the dense scaling config). */
static double normal01_t(orc_mt64* g) {
  const double u1 = orc_uniform_unit(g), u2 = orc_uniform_unit(g);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
}

int orc_gen_tiled(size_t m, size_t n, size_t r, uint64_t seed, size_t T, double* x) {
  if (T == 0) T = 4096;
  const size_t nbi = (m + T - 1) / T, nbj = (n + T - 1) / T;
  double* w = (double*)malloc(sizeof(double) * m * r);
  double* h = (double*)malloc(sizeof(double) * r * n);
  if (!w || !h) { free(w); free(h); return ENMF_INVALID_ARGUMENT; }
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_orc_threads)
  for (size_t bi = 0; bi < nbi; ++bi) {
    orc_mt64 g;
    orc_mt64_seed(&g, orc_mix_seed(seed, 1, bi));
    const size_t i1 = (bi + 1) * T < m ? (bi + 1) * T : m;
    for (size_t i = bi * T; i < i1; ++i)
      for (size_t k = 0; k < r; ++k) w[i * r + k] = orc_uniform_unit(&g);
  }
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_orc_threads)
  for (size_t bj = 0; bj < nbj; ++bj) {
    orc_mt64 g;
    orc_mt64_seed(&g, orc_mix_seed(seed, 2, bj));
    const size_t j1 = (bj + 1) * T < n ? (bj + 1) * T : n;
    for (size_t k = 0; k < r; ++k)
      for (size_t j = bj * T; j < j1; ++j) h[k * n + j] = orc_uniform_unit(&g);
  }
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_orc_threads)
  for (size_t t = 0; t < nbi * nbj; ++t) {
    const size_t bi = t / nbj, bj = t % nbj;
    const size_t i0 = bi * T, i1 = i0 + T < m ? i0 + T : m;
    const size_t j0 = bj * T, j1 = j0 + T < n ? j0 + T : n;
    for (size_t i = i0; i < i1; ++i) {
      double* xi = x + i * n;
      for (size_t j = j0; j < j1; ++j) xi[j] = 0.0;
      for (size_t k = 0; k < r; ++k) {
        const double wik = w[i * r + k];
        const double* hk = h + k * n;
        for (size_t j = j0; j < j1; ++j) xi[j] += wik * hk[j];
      }
    }
    orc_mt64 g;
    orc_mt64_seed(&g, orc_mix_seed(seed, 3, t));
    for (size_t i = i0; i < i1; ++i)
      for (size_t j = j0; j < j1; ++j) x[i * n + j] += 0.01 * fabs(normal01_t(&g));
  }
  free(w);
  free(h);
  return ENMF_OK;
}

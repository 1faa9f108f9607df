/*
 * enmf_oracle.c — CPU restatement of the reference enmf hot path (plain C11).
 *
 * TEST INFRASTRUCTURE ONLY (see enmf_oracle.h).  Each function cites the
 * reference function it restates (paths relative to /root/reference/proj/include/enmf).
 * The floating-point operation order of every reduction is the reference's, so
 * that with -ffp-contract=off the results are bitwise identical to the reference
 * (checked against oracle/_ref in tests/test_oracle.py).
 *
 * The synthetic-data generators at the bottom (orc_gen_c2/c3/c5/docs) are NOT in
 * the reference: they realise the BASELINE.json config descriptions with a fixed
 * documented draw order on one mt19937_64 stream.
 */
#define _POSIX_C_SOURCE 199309L
#include "enmf_oracle.h"

#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[512];
/* Multi-threaded bit-exact replica kernels (replica.c); used when orc_set_threads(n > 1). */
extern int g_orc_threads;
void rep_cross_wx(const double* w, const double* x, size_t m, size_t n, size_t r, double* out);
void rep_cross_xht(const double* x, const double* h, size_t m, size_t n, size_t r, double* out);
void rep_gram(const double* a, size_t rows, size_t r, double* g);
void rep_gram_rows(const double* t, size_t r, size_t n, double* g);
int rep_hals_solve(const double* gram, const double* cross, const double* h0, size_t r, size_t n,
                   uint64_t max_sweeps, double stall_fraction, double* h, int32_t* sweeps);

static void set_err(const char* msg) { snprintf(g_err, sizeof g_err, "%s", msg); }
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ rng.hpp */
/* std::mt19937_64 (the standard's published parameters). */
void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  g->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  static const uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (g->mt[i] & kUpper) | (g->mt[(i + 1) % 312] & kLower);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* rng.hpp:30-34 */
uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* rng.hpp:38-44 */
uint64_t orc_mix_seed(uint64_t base, uint64_t a, uint64_t b) {
  const uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
  uint64_t h = orc_mix64(base + kGolden);
  h = orc_mix64(h ^ (a + kGolden));
  h = orc_mix64(h ^ (b + kGolden));
  return h;
}

/* rng.hpp:47-49 */
double orc_uniform_unit(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }

static void fill_uniform(double* p, size_t count, orc_mt64* g) {  /* rng.hpp:52-55 */
  for (size_t i = 0; i < count; ++i) p[i] = orc_uniform_unit(g);
}

/* --------------------------------------------------------------- linalg.hpp */
/* Neumaier CompensatedSum, linalg.hpp:27-44 */
typedef struct { double sum, c; } csum;
static void cs_add(csum* s, double v) {
  const double t = s->sum + v;
  if (fabs(s->sum) >= fabs(v)) {
    s->c += (s->sum - t) + v;
  } else {
    s->c += (v - t) + s->sum;
  }
  s->sum = t;
}
static double cs_value(const csum* s) { return s->sum + s->c; }

/* multiply, linalg.hpp:174-189 (ikj) */
static void multiply(const double* a, const double* b, size_t m, size_t k, size_t n, double* out) {
  memset(out, 0, sizeof(double) * m * n);
  for (size_t i = 0; i < m; ++i) {
    double* oi = out + i * n;
    for (size_t p = 0; p < k; ++p) {
      const double aip = a[i * k + p];
      const double* bp = b + p * n;
      for (size_t j = 0; j < n; ++j) oi[j] += aip * bp[j];
    }
  }
}

/* gram, linalg.hpp:49-64: upper triangle accumulated over rows i, mirrored. */
void orc_gram(const double* a, size_t m, size_t r, double* g) {
  memset(g, 0, sizeof(double) * r * r);
  for (size_t i = 0; i < m; ++i) {
    const double* ai = a + i * r;
    for (size_t k = 0; k < r; ++k) {
      const double aik = ai[k];
      double* gk = g + k * r;
      for (size_t j = k; j < r; ++j) gk[j] += aik * ai[j];
    }
  }
  for (size_t k = 0; k < r; ++k)
    for (size_t j = k + 1; j < r; ++j) g[j * r + k] = g[k * r + j];
}

/* gram(tᵀ) for t r×n, without materialising the transpose (the transpose is
 * exact, and gram iterates the rows of tᵀ = the columns of t in order). */
void orc_gram_rows(const double* t, size_t r, size_t n, double* g) {
  memset(g, 0, sizeof(double) * r * r);
  for (size_t i = 0; i < n; ++i) {
    for (size_t k = 0; k < r; ++k) {
      const double aik = t[k * n + i];
      double* gk = g + k * r;
      for (size_t j = k; j < r; ++j) gk[j] += aik * t[j * n + i];
    }
  }
  for (size_t k = 0; k < r; ++k)
    for (size_t j = k + 1; j < r; ++j) g[j * r + k] = g[k * r + j];
}

/* cross_wx dense, linalg.hpp:67-83 */
void orc_cross_wx(const double* w, const double* x, size_t m, size_t n, size_t r, double* out) {
  memset(out, 0, sizeof(double) * r * n);
  for (size_t i = 0; i < m; ++i) {
    const double* wi = w + i * r;
    const double* xi = x + i * n;
    for (size_t k = 0; k < r; ++k) {
      const double wik = wi[k];
      double* ok = out + k * n;
      for (size_t j = 0; j < n; ++j) ok[j] += wik * xi[j];
    }
  }
}

/* cross_wx CSR, linalg.hpp:86-104 */
void orc_cross_wx_csr(const double* w, const uint64_t* off, const uint64_t* cidx, const double* v,
                      size_t m, size_t n, size_t r, double* out) {
  memset(out, 0, sizeof(double) * r * n);
  for (size_t i = 0; i < m; ++i) {
    const double* wi = w + i * r;
    for (uint64_t p = off[i]; p < off[i + 1]; ++p) {
      const size_t j = (size_t)cidx[p];
      const double val = v[p];
      for (size_t k = 0; k < r; ++k) out[k * n + j] += wi[k] * val;
    }
  }
}

/* cross_xht dense, linalg.hpp:107-124 */
void orc_cross_xht(const double* x, const double* h, size_t m, size_t n, size_t r, double* out) {
  for (size_t i = 0; i < m; ++i) {
    const double* xi = x + i * n;
    double* oi = out + i * r;
    for (size_t k = 0; k < r; ++k) {
      const double* hk = h + k * n;
      double s = 0.0;
      for (size_t j = 0; j < n; ++j) s += xi[j] * hk[j];
      oi[k] = s;
    }
  }
}

/* cross_xht CSR, linalg.hpp:127-146 */
void orc_cross_xht_csr(const uint64_t* off, const uint64_t* cidx, const double* v, const double* h,
                       size_t m, size_t n, size_t r, double* out) {
  memset(out, 0, sizeof(double) * m * r);
  for (size_t i = 0; i < m; ++i) {
    double* oi = out + i * r;
    for (uint64_t p = off[i]; p < off[i + 1]; ++p) {
      const size_t j = (size_t)cidx[p];
      const double val = v[p];
      for (size_t k = 0; k < r; ++k) oi[k] += val * h[k * n + j];
    }
  }
}

/* frob_norm_sq, linalg.hpp:160-171 */
double orc_frob_norm_sq(const double* x, size_t count) {
  csum s = {0.0, 0.0};
  for (size_t i = 0; i < count; ++i) cs_add(&s, x[i] * x[i]);
  return cs_value(&s);
}

/* fast_error, engine.hpp:121-136 */
double orc_fast_error(double norm_x_sq, const double* w, const double* xht, const double* hht,
                      size_t m, size_t r) {
  csum acc = {0.0, 0.0};
  cs_add(&acc, norm_x_sq);
  for (size_t i = 0; i < m * r; ++i) cs_add(&acc, -2.0 * w[i] * xht[i]);
  double* wtw = (double*)malloc(sizeof(double) * r * r);
  if (g_orc_threads > 1) rep_gram(w, m, r, wtw);
  else orc_gram(w, m, r, wtw);
  for (size_t i = 0; i < r * r; ++i) cs_add(&acc, wtw[i] * hht[i]);
  free(wtw);
  const double v = cs_value(&acc);
  return sqrt(v > 0.0 ? v : 0.0);  /* std::max(0.0, v) = (0.0 < v) ? v : 0.0; NaN -> 0 */
}

/* ----------------------------------------------------------------- nnls.hpp */
static double max_diagonal(const double* g, size_t r) {  /* nnls.hpp:99-103 */
  double m = 0.0;
  for (size_t i = 0; i < r; ++i) m = (m < g[i * r + i]) ? g[i * r + i] : m;
  return m;
}

/* InnerLoopPolicy::derive, nnls.hpp:79-87 */
uint64_t orc_derive_max_sweeps(double setup_flops, double sweep_flops, double ratio) {
  const double rho = sweep_flops > 0.0 ? setup_flops / sweep_flops : 0.0;
  return 1 + (uint64_t)floor(ratio * rho);
}

/* hals_row_update_impl, nnls.hpp:111-136.  h is r×n row-major. */
static int hals_row_update(const double* gram, const double* cross, double* h, size_t r, size_t n,
                           size_t k, double floor_, double* scratch, double* gain_out) {
  const double gkk = gram[k * r + k];
  if (!(gkk > floor_)) return -1;
  memcpy(scratch, cross + k * n, sizeof(double) * n);
  for (size_t j = 0; j < r; ++j) {
    if (j == k) continue;
    const double gkj = gram[k * r + j];
    if (gkj == 0.0) continue;
    const double* hj = h + j * n;
    for (size_t t = 0; t < n; ++t) scratch[t] -= gkj * hj[t];
  }
  double* hk = h + k * n;
  double gain = 0.0;
  for (size_t t = 0; t < n; ++t) {
    const double target = scratch[t] / gkk;
    const double next = target > 0.0 ? target : 0.0;
    const double d_old = hk[t] - target;
    const double d_new = next - target;
    gain += d_old * d_old - d_new * d_new;
    hk[t] = next;
  }
  *gain_out = gkk * gain;
  return 0;
}

/* hals_solve, nnls.hpp:154-176 */
int orc_hals_solve(const double* gram, const double* cross, const double* h0, size_t r, size_t n,
                   uint64_t max_sweeps, double stall_fraction, double* h, int32_t* sweeps) {
  if (max_sweeps < 1) { set_err("InnerLoopPolicy: max_sweeps must be >= 1"); return ENMF_INVALID_ARGUMENT; }
  for (size_t i = 0; i < r * n; ++i)
    if (!isfinite(h0[i])) { set_err("hals_solve: warm start must be finite"); return ENMF_INVALID_ARGUMENT; }
  const double floor_ = 1e-16 * max_diagonal(gram, r);
  if (h != h0) memcpy(h, h0, sizeof(double) * r * n);
  double* scratch = (double*)malloc(sizeof(double) * n);
  double first_gain = 0.0;
  int rc = ENMF_OK;
  uint64_t sweep;
  for (sweep = 1;; ++sweep) {
    double gain = 0.0;
    for (size_t k = 0; k < r; ++k) {
      double gk;
      if (hals_row_update(gram, cross, h, r, n, k, floor_, scratch, &gk) != 0) {
        char msg[96];
        snprintf(msg, sizeof msg, "near-zero Gram diagonal at index %zu", k);
        set_err(msg);
        rc = ENMF_DEGENERATE_COLUMN;
        goto out;
      }
      gain += gk;
    }
    if (sweep == 1) first_gain = gain;
    if (sweep >= max_sweeps) break;
    if (gain <= stall_fraction * (first_gain < 0.0 ? 0.0 : first_gain)) break;
  }
out:
  free(scratch);
  if (sweeps) *sweeps = (int32_t)sweep;
  return rc;
}

/* cholesky, nnls.hpp:215-229 */
static size_t cholesky(double* a, size_t f, double pivot_floor) {
  for (size_t j = 0; j < f; ++j) {
    double d = a[j * f + j];
    for (size_t p = 0; p < j; ++p) d -= a[j * f + p] * a[j * f + p];
    if (!(d > pivot_floor)) return j;
    const double ljj = sqrt(d);
    a[j * f + j] = ljj;
    for (size_t i = j + 1; i < f; ++i) {
      double s = a[i * f + j];
      for (size_t p = 0; p < j; ++p) s -= a[i * f + p] * a[j * f + p];
      a[i * f + j] = s / ljj;
    }
  }
  return f;
}

/* cholesky_solve, nnls.hpp:232-243 */
static void cholesky_solve(const double* l, size_t f, double* b) {
  for (size_t i = 0; i < f; ++i) {
    double s = b[i];
    for (size_t p = 0; p < i; ++p) s -= l[i * f + p] * b[p];
    b[i] = s / l[i * f + i];
  }
  for (size_t ii = f; ii-- > 0;) {
    double s = b[ii];
    for (size_t p = ii + 1; p < f; ++p) s -= l[p * f + ii] * b[p];
    b[ii] = s / l[ii * f + ii];
  }
}

/* active_set_solve, nnls.hpp:259-406, restated per column.  The reference
 * groups columns with equal passive sets to share one factorization; the
 * factorization, the pivot-drop/ban decisions and hence every per-column result
 * are functions of the passive set alone, so solving each column on its own is
 * identical.  The exchange limit 3·r·n is a global count; it trips
 * iff the total exchange count exceeds it, independent of processing order. */
/* cmax_all / n_all: max|cross| and column count of the WHOLE problem when this call solves a
 * shard of its columns (the sharded model, oracle/sharded_model.py); < 0 / 0 = this call's own. */
int orc_active_set_solve_shard(const double* gram, const double* cross, const double* h0, size_t r, size_t n,
                               double cmax_all, size_t n_all, double* h, int32_t* rounds, uint64_t* exch_out) {
  for (size_t i = 0; i < r * n; ++i)
    if (!isfinite(h0[i])) { set_err("active_set_solve: warm start must be finite"); return ENMF_INVALID_ARGUMENT; }
  double cmax = 0.0;
  for (size_t i = 0; i < r * n; ++i) cmax = (cmax < fabs(cross[i])) ? fabs(cross[i]) : cmax;
  if (cmax_all >= 0.0) cmax = cmax_all;
  const double feas_tol = 1e-12 * (1.0 + cmax);
  const double pivot_floor = 1e-12 * max_diagonal(gram, r);
  const uint64_t exchange_limit = 3ULL * r * (n_all ? n_all : n);
  uint64_t exchanges = 0;
  int32_t max_rounds = 0;

  unsigned char* passive = (unsigned char*)malloc(r);
  unsigned char* banned = (unsigned char*)malloc(r);
  size_t* fidx = (size_t*)malloc(sizeof(size_t) * r);
  size_t* infeas = (size_t*)malloc(sizeof(size_t) * 2 * r);
  double* cff = (double*)malloc(sizeof(double) * r * r);
  double* lfac = (double*)malloc(sizeof(double) * r * r);
  double* df = (double*)malloc(sizeof(double) * r);
  double* xf = (double*)malloc(sizeof(double) * r);
  double* resid = (double*)malloc(sizeof(double) * r);
  int rc = ENMF_OK;

  memset(h, 0, sizeof(double) * r * n);
  for (size_t col = 0; col < n && rc == ENMF_OK; ++col) {
    for (size_t i = 0; i < r; ++i) { passive[i] = h0[i * n + col] > 0.0 ? 1 : 0; banned[i] = 0; }
    int best_inf = INT_MAX, backup = 3;
    int32_t solves = 0;
    for (;;) {
      ++solves;
      size_t f = 0;
      for (size_t i = 0; i < r; ++i) if (passive[i]) fidx[f++] = i;
      for (;;) {
        if (f == 0) break;
        for (size_t a = 0; a < f; ++a)
          for (size_t b = 0; b < f; ++b) cff[a * f + b] = gram[fidx[a] * r + fidx[b]];
        memcpy(lfac, cff, sizeof(double) * f * f);
        const size_t bad = cholesky(lfac, f, pivot_floor);
        if (bad == f) break;
        const size_t var = fidx[bad];
        passive[var] = 0;
        banned[var] = 1;
        for (size_t a = bad; a + 1 < f; ++a) fidx[a] = fidx[a + 1];
        --f;
      }
      for (size_t a = 0; a < f; ++a) df[a] = cross[fidx[a] * n + col];
      memcpy(xf, df, sizeof(double) * f);
      if (f > 0) {
        cholesky_solve(lfac, f, xf);
        for (size_t a = 0; a < f; ++a) {
          double s = df[a];
          for (size_t b = 0; b < f; ++b) s -= cff[a * f + b] * xf[b];
          resid[a] = s;
        }
        cholesky_solve(lfac, f, resid);
        for (size_t a = 0; a < f; ++a) xf[a] += resid[a];
      }
      size_t ni = 0;
      for (size_t a = 0; a < f; ++a) if (xf[a] < -feas_tol) infeas[ni++] = fidx[a];
      for (size_t i = 0; i < r; ++i) {
        if (passive[i] || banned[i]) continue;
        double y = -cross[i * n + col];
        for (size_t a = 0; a < f; ++a) y += gram[i * r + fidx[a]] * xf[a];
        if (y < -feas_tol) infeas[ni++] = i;
      }
      if (ni == 0) {
        for (size_t a = 0; a < f; ++a) h[fidx[a] * n + col] = xf[a] > 0.0 ? xf[a] : 0.0;
        break;
      }
      if (++exchanges > exchange_limit) {
        char msg[128];
        snprintf(msg, sizeof msg, "active_set_solve: exchange limit of %llu rounds exceeded",
                 (unsigned long long)exchange_limit);
        set_err(msg);
        rc = ENMF_NO_CONVERGENCE;
        break;
      }
      const int count = (int)ni;
      if (count < best_inf) {
        best_inf = count;
        backup = 3;
        for (size_t q = 0; q < ni; ++q) passive[infeas[q]] ^= 1;
      } else if (backup > 0) {
        --backup;
        for (size_t q = 0; q < ni; ++q) passive[infeas[q]] ^= 1;
      } else {
        size_t v = infeas[0];
        for (size_t q = 1; q < ni; ++q) v = infeas[q] > v ? infeas[q] : v;
        passive[v] ^= 1;
      }
    }
    if (solves > max_rounds) max_rounds = solves;
  }
  free(passive); free(banned); free(fidx); free(infeas); free(cff); free(lfac);
  free(df); free(xf); free(resid);
  if (rounds) *rounds = max_rounds;
  if (exch_out) *exch_out = exchanges;
  return rc;
}

/* active_set_solve, nnls.hpp:259-406 */
int orc_active_set_solve(const double* gram, const double* cross, const double* h0, size_t r,
                         size_t n, double* h, int32_t* rounds) {
  return orc_active_set_solve_shard(gram, cross, h0, r, n, -1.0, 0, h, rounds, NULL);
}

/* `count` uniform_unit draws (rng.hpp:47-49) of mt19937_64(seed) — the reinit stream */
void orc_uniform_stream(uint64_t seed, size_t count, double* out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  for (size_t i = 0; i < count; ++i) out[i] = orc_uniform_unit(&g);
}

/* --------------------------------------------------------------- engine.hpp */
/* update_beta, engine.hpp:88-99 */
enmf_gpu_beta_schedule orc_update_beta(enmf_gpu_beta_schedule s, int error_decreased) {
  const double used = s.beta;
  if (error_decreased) {
    const double g = s.gamma * s.beta;
    s.beta = (g < s.beta_bar) ? g : s.beta_bar;                  /* std::min(beta_bar, gamma*beta) */
    const double gb = s.gamma_bar * s.beta_bar;
    s.beta_bar = (gb < 1.0) ? gb : 1.0;                         /* std::min(1.0, ...) */
  } else {
    s.beta = s.beta / s.eta;
    s.beta_bar = s.beta_prev;
  }
  s.beta_prev = used;
  return s;
}

/* SolverConfig::validate, engine.hpp:175-199 (+ BetaSchedule::validate :71-81) */
int orc_config_validate(const enmf_gpu_config* c) {
  if (c->hp != 1 && c->hp != 2 && c->hp != 3) { set_err("SolverConfig: hp must be 1, 2 or 3"); return ENMF_INVALID_ARGUMENT; }
  if (!(c->beta0 >= 0.0) || !(c->beta0 < 1.0)) { set_err("SolverConfig: beta0 must lie in [0, 1)"); return ENMF_INVALID_ARGUMENT; }
  if (c->extrapolation_enabled && c->beta0 > 0.0) {
    /* BetaSchedule{beta=beta0, beta_bar=1, beta_prev=beta0}.validate() */
    if (!(c->beta0 >= 0.0) || !(1.0 <= 1.0) || !(c->beta0 <= 1.0)) { set_err("BetaSchedule: need 0 <= beta <= beta_bar <= 1"); return ENMF_INVALID_ARGUMENT; }
    if (!(1.0 < c->gamma_bar) || !(c->gamma_bar < c->gamma) || !(c->gamma < c->eta)) {
      set_err("BetaSchedule: need 1 < gamma_bar < gamma < eta");
      return ENMF_INVALID_ARGUMENT;
    }
  }
  if (!(c->max_seconds > 0.0)) { set_err("SolverConfig: max_seconds must be > 0"); return ENMF_INVALID_ARGUMENT; }
  if (!(c->inner_sweep_ratio > 0.0)) { set_err("SolverConfig: inner_sweep_ratio must be > 0"); return ENMF_INVALID_ARGUMENT; }
  if (!(c->inner_stall_fraction > 0.0) || c->inner_stall_fraction >= 1.0) {
    set_err("SolverConfig: inner_stall_fraction must lie in (0, 1)");
    return ENMF_INVALID_ARGUMENT;
  }
  if (c->inner_h != ENMF_INNER_EXACT && c->inner_h != ENMF_INNER_HALS) { set_err("SolverConfig: bad inner_h"); return ENMF_INVALID_ARGUMENT; }
  if (c->inner_w != ENMF_INNER_EXACT && c->inner_w != ENMF_INNER_HALS) { set_err("SolverConfig: bad inner_w"); return ENMF_INVALID_ARGUMENT; }
  return ENMF_OK;
}

/* Data matrix: dense row-major or CSR (the two MatrixX instantiations). */
typedef struct {
  int sparse;
  const double* x;
  const uint64_t* off; const uint64_t* cidx; const double* vals;
  size_t m, n, nnz;
} xmat;

static void x_cross_wx(const xmat* X, const double* w, size_t r, double* out) {
  if (!X->sparse && g_orc_threads > 1) rep_cross_wx(w, X->x, X->m, X->n, r, out);
  else if (X->sparse) orc_cross_wx_csr(w, X->off, X->cidx, X->vals, X->m, X->n, r, out);
  else orc_cross_wx(w, X->x, X->m, X->n, r, out);
}
static void x_cross_xht(const xmat* X, const double* h, size_t r, double* out) {
  if (!X->sparse && g_orc_threads > 1) rep_cross_xht(X->x, h, X->m, X->n, r, out);
  else if (X->sparse) orc_cross_xht_csr(X->off, X->cidx, X->vals, h, X->m, X->n, r, out);
  else orc_cross_xht(X->x, h, X->m, X->n, r, out);
}

static void transpose(const double* a, size_t rows, size_t cols, double* t) {
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < cols; ++j) t[j * rows + i] = a[i * cols + j];
}

static int all_finite(const double* a, size_t count) {
  for (size_t i = 0; i < count; ++i) if (!isfinite(a[i])) return 0;
  return 1;
}

/* extrapolate, engine.hpp:102-113; clamp_nonnegative matrix.hpp:114-116 */
static void extrapolate(const double* next, const double* prev, double beta, size_t count,
                        int clamp, double* out) {
  for (size_t i = 0; i < count; ++i) {
    double v = next[i] + beta * (next[i] - prev[i]);
    out[i] = clamp ? (v > 0.0 ? v : 0.0) : v;
  }
}

/* reinit_columns + gram_with_reinit, engine.hpp:268-296, for a factor held as
 * `a` with `rows` rows and r columns, where column c of the reference matrix is
 * the strided sequence a[c*cs + i*rs], i = 0..rows-1.  Computes g = gram. */
static int gram_with_reinit(double* a, size_t rows, size_t r, size_t rs, size_t cs,
                            uint64_t reinit_seed, uint64_t salt, int* modified, double* g) {
  size_t* bad = (size_t*)malloc(sizeof(size_t) * (r ? r : 1));
  for (uint64_t attempt = 0;; ++attempt) {
    if (g_orc_threads > 1 && cs == 1 && rs == r) {
      rep_gram(a, rows, r, g);
    } else if (g_orc_threads > 1 && rs == 1 && cs == rows) {
      rep_gram_rows(a, r, rows, g);
    } else {
      memset(g, 0, sizeof(double) * r * r);
      for (size_t i = 0; i < rows; ++i)
        for (size_t k = 0; k < r; ++k) {
          const double aik = a[k * cs + i * rs];
          for (size_t j = k; j < r; ++j) g[k * r + j] += aik * a[j * cs + i * rs];
        }
      for (size_t k = 0; k < r; ++k)
        for (size_t j = k + 1; j < r; ++j) g[j * r + k] = g[k * r + j];
    }
    const double floor_ = 1e-16 * max_diagonal(g, r);
    size_t nb = 0;
    for (size_t k = 0; k < r; ++k) if (!(g[k * r + k] > floor_)) bad[nb++] = k;
    if (nb == 0) { free(bad); return ENMF_OK; }
    if (attempt > r + 2) {
      set_err("degenerate factor column persists after reinitialization");
      free(bad);
      return ENMF_NO_CONVERGENCE;
    }
    orc_mt64 gen;
    orc_mt64_seed(&gen, orc_mix_seed(reinit_seed, salt, attempt));
    for (size_t q = 0; q < nb; ++q)
      for (size_t i = 0; i < rows; ++i) a[bad[q] * cs + i * rs] = orc_uniform_unit(&gen);
    if (modified) *modified = 1;
  }
}

/* hals_solve through the replica when threaded; the replica reports the degenerate row
 * without the message, so the port's solver reruns to produce it (same result). */
static int hals(const double* gram, const double* cross, const double* h0, size_t r, size_t n,
                uint64_t max_sweeps, double stall_fraction, double* h, int32_t* sweeps) {
  if (g_orc_threads > 1 && r <= 4096) {
    int rc = rep_hals_solve(gram, cross, h0, r, n, max_sweeps, stall_fraction, h, sweeps);
    if (rc != ENMF_DEGENERATE_COLUMN) return rc;
  }
  return orc_hals_solve(gram, cross, h0, r, n, max_sweeps, stall_fraction, h, sweeps);
}

typedef struct {
  double *w, *h, *w_y, *h_y, *w_n, *h_n;
  double err_prev;
  enmf_gpu_beta_schedule schedule;
  int restarted;
} ext_state;

/* step, engine.hpp:309-440 */
static int step(const xmat* X, double norm_x_sq, ext_state* st, const enmf_gpu_config* cfg,
                size_t r, uint64_t iteration, enmf_gpu_iter* rec, double* ws) {
  const size_t m = X->m, n = X->n;
  const double beta = cfg->extrapolation_enabled ? st->schedule.beta : 0.0;
  const double setup_flops = X->sparse ? (double)X->nnz * (double)r : (double)m * (double)n * (double)r;
  double* gram_h = ws;                 /* r×r */
  double* gram_t = gram_h + r * r;     /* r×r */
  double* cross_h = gram_t + r * r;    /* r×n */
  double* xht = cross_h + r * n;       /* m×r */
  double* pw_cross = xht + m * r;      /* r×m */
  double* wy_t = pw_cross + r * m;     /* r×m */
  double* wn_t = wy_t + r * m;         /* r×m */
  double* lit_g = wn_t + r * m;        /* r×r */
  double* lit_x = lit_g + r * r;       /* m×r */
  int rc;
  memset(rec, 0, sizeof *rec);
  rec->iteration = iteration;
  rec->beta = beta;

  /* H update (:323-333) */
  int mod = 0;
  rc = gram_with_reinit(st->w_y, m, r, r, 1, cfg->reinit_seed, 2 * iteration, &mod, gram_h);
  if (rc) return rc;
  if (mod) rec->reinit_events |= 1;
  x_cross_wx(X, st->w_y, r, cross_h);
  if (cfg->inner_h == ENMF_INNER_EXACT) {
    rc = orc_active_set_solve(gram_h, cross_h, st->h_y, r, n, st->h_n, &rec->inner_h_count);
  } else {
    uint64_t ms = cfg->inner_max_sweeps ? cfg->inner_max_sweeps
                  : orc_derive_max_sweeps(setup_flops, (double)n * (double)r * (double)r, cfg->inner_sweep_ratio);
    rc = hals(gram_h, cross_h, st->h_y, r, n, ms, cfg->inner_stall_fraction, st->h_n,
              &rec->inner_h_count);
  }
  if (rc) return rc;
  if (!all_finite(st->h_n, r * n)) { set_err("H update produced a non-finite value"); return ENMF_NON_FINITE; }

  /* early H extrapolation (:340-347) */
  if (cfg->hp >= 2) {
    if (cfg->extrapolation_enabled) extrapolate(st->h_n, st->h, beta, r * n, cfg->hp == 3, st->h_y);
    else memcpy(st->h_y, st->h_n, sizeof(double) * r * n);
  }
  const int w_target_is_hy = cfg->hp >= 2 || (cfg->literal_hp1_order && cfg->extrapolation_enabled);

  /* W update (:353-379) */
  double* target = w_target_is_hy ? st->h_y : st->h_n;
  mod = 0;
  rc = gram_with_reinit(target, n, r, 1, n, cfg->reinit_seed, 2 * iteration + 1, &mod, gram_t);
  if (rc) return rc;
  if (mod) rec->reinit_events |= 2;
  x_cross_xht(X, target, r, xht);
  transpose(xht, m, r, pw_cross);
  transpose(st->w_y, m, r, wy_t);
  if (cfg->inner_w == ENMF_INNER_EXACT) {
    rc = orc_active_set_solve(gram_t, pw_cross, wy_t, r, m, wn_t, &rec->inner_w_count);
  } else {
    uint64_t ms = cfg->inner_max_sweeps ? cfg->inner_max_sweeps
                  : orc_derive_max_sweeps(setup_flops, (double)m * (double)r * (double)r, cfg->inner_sweep_ratio);
    rc = hals(gram_t, pw_cross, wy_t, r, m, ms, cfg->inner_stall_fraction, wn_t,
              &rec->inner_w_count);
  }
  if (rc) return rc;
  transpose(wn_t, r, m, st->w_n);
  if (!all_finite(st->w_n, m * r)) { set_err("W update produced a non-finite value"); return ENMF_NON_FINITE; }

  /* W extrapolation and late H extrapolation (:386-397) */
  if (cfg->extrapolation_enabled) extrapolate(st->w_n, st->w, beta, m * r, 0, st->w_y);
  else memcpy(st->w_y, st->w_n, sizeof(double) * m * r);
  if (cfg->hp == 1) {
    if (cfg->extrapolation_enabled) extrapolate(st->h_n, st->h, beta, r * n, 0, st->h_y);
    else memcpy(st->h_y, st->h_n, sizeof(double) * r * n);
  }

  /* error (:402-416) */
  double err;
  if (cfg->hp == 1 && cfg->literal_hp1_order && cfg->extrapolation_enabled) {
    if (g_orc_threads > 1) rep_gram_rows(st->h_y, r, n, lit_g);
    else orc_gram_rows(st->h_y, r, n, lit_g);
    x_cross_xht(X, st->h_y, r, lit_x);
    err = orc_fast_error(norm_x_sq, st->w_n, lit_x, lit_g, m, r);
  } else {
    err = orc_fast_error(norm_x_sq, st->w_n, xht, gram_t, m, r);
  }
  if (!isfinite(err)) { set_err("error evaluation produced a non-finite value"); return ENMF_NON_FINITE; }

  /* restart / accept (:420-434) */
  if (err > st->err_prev) {
    memcpy(st->w_y, st->w, sizeof(double) * m * r);
    memcpy(st->h_y, st->h, sizeof(double) * r * n);
    st->restarted = 1;
  } else {
    memcpy(st->w, st->w_n, sizeof(double) * m * r);
    memcpy(st->h, st->h_n, sizeof(double) * r * n);
    st->restarted = 0;
  }
  rec->restarted = st->restarted;
  if (cfg->extrapolation_enabled) st->schedule = orc_update_beta(st->schedule, err <= st->err_prev);
  st->err_prev = err;
  rec->error = err;
  const double norm_x = sqrt(norm_x_sq);
  rec->relative_error = norm_x > 0.0 ? err / norm_x : 0.0;
  return ENMF_OK;
}

/* run, engine.hpp:447-521 (elapsed fields written as 0: TimingMode::none). */
static int run_impl(const xmat* X, const double* w0, const double* h0, size_t r,
                    const enmf_gpu_config* cfg, enmf_gpu_iter* iters, size_t iters_cap,
                    size_t* n_iters, double* w_out, double* h_out, double* norm_x_out) {
  int rc = orc_config_validate(cfg);
  if (rc) return rc;
  const size_t m = X->m, n = X->n;
  if (m == 0 || n == 0 || r == 0) { set_err("run: empty shape"); return ENMF_INVALID_ARGUMENT; }
  for (size_t i = 0; i < m * r; ++i)
    if (!isfinite(w0[i]) || !(w0[i] >= 0.0)) { set_err("run: initial factors must be finite and nonnegative"); return ENMF_INVALID_ARGUMENT; }
  for (size_t i = 0; i < r * n; ++i)
    if (!isfinite(h0[i]) || !(h0[i] >= 0.0)) { set_err("run: initial factors must be finite and nonnegative"); return ENMF_INVALID_ARGUMENT; }

  const double norm_x_sq = X->sparse ? orc_frob_norm_sq(X->vals, X->nnz) : orc_frob_norm_sq(X->x, m * n);
  const double norm_x = sqrt(norm_x_sq);
  if (norm_x_out) *norm_x_out = norm_x;

  ext_state st;
  const size_t wsz = m * r, hsz = r * n;
  st.w = (double*)malloc(sizeof(double) * wsz); st.w_y = (double*)malloc(sizeof(double) * wsz);
  st.w_n = (double*)malloc(sizeof(double) * wsz);
  st.h = (double*)malloc(sizeof(double) * hsz); st.h_y = (double*)malloc(sizeof(double) * hsz);
  st.h_n = (double*)malloc(sizeof(double) * hsz);
  memcpy(st.w, w0, sizeof(double) * wsz); memcpy(st.w_y, w0, sizeof(double) * wsz);
  memcpy(st.h, h0, sizeof(double) * hsz); memcpy(st.h_y, h0, sizeof(double) * hsz);
  memset(st.w_n, 0, sizeof(double) * wsz); memset(st.h_n, 0, sizeof(double) * hsz);
  st.schedule.beta = cfg->beta0; st.schedule.beta_bar = 1.0; st.schedule.beta_prev = cfg->beta0;
  st.schedule.gamma = cfg->gamma; st.schedule.gamma_bar = cfg->gamma_bar; st.schedule.eta = cfg->eta;
  st.restarted = 0;
  double* ws = (double*)malloc(sizeof(double) * (4 * r * r + r * n + 5 * m * r));

  /* e(0) (:487-503) */
  {
    double* g0 = ws;
    double* x0 = ws + r * r;
    if (g_orc_threads > 1) rep_gram_rows(h0, r, n, g0);
    else orc_gram_rows(h0, r, n, g0);
    x_cross_xht(X, h0, r, x0);
    const double e0 = orc_fast_error(norm_x_sq, w0, x0, g0, m, r);
    st.err_prev = e0;
    size_t cnt = 0;
    if (iters_cap > 0) {
      memset(&iters[0], 0, sizeof iters[0]);
      iters[0].iteration = 0;
      iters[0].error = e0;
      iters[0].relative_error = norm_x > 0.0 ? e0 / norm_x : 0.0;
      iters[0].beta = cfg->extrapolation_enabled ? cfg->beta0 : 0.0;
      cnt = 1;
    }
    for (uint64_t k = 1; k <= cfg->max_outer_iterations; ++k) {
      enmf_gpu_iter rec;
      rc = step(X, norm_x_sq, &st, cfg, r, k, &rec, ws);
      if (rc) break;
      if (cnt < iters_cap) iters[cnt] = rec;
      ++cnt;
    }
    if (n_iters) *n_iters = cnt;
  }
  if (rc == ENMF_OK) {
    if (w_out) memcpy(w_out, st.w, sizeof(double) * wsz);
    if (h_out) memcpy(h_out, st.h, sizeof(double) * hsz);
  }
  free(ws); free(st.w); free(st.w_y); free(st.w_n); free(st.h); free(st.h_y); free(st.h_n);
  return rc;
}

/* run()'s prologue then `nsteps` step() calls; *seconds = time inside step()
 * only (bench.py cpu_baseline when oracle/_ref is absent). */

int orc_time_steps(const double* x, size_t m, size_t n, const double* w0, const double* h0, size_t r,
                   const enmf_gpu_config* cfg, size_t nsteps, double* seconds, double* last_rel_err) {
  int rc = orc_config_validate(cfg);
  if (rc) return rc;
  xmat X = {0, x, NULL, NULL, NULL, m, n, m * n};
  const double nx2 = orc_frob_norm_sq(x, m * n);
  ext_state st;
  const size_t wsz = m * r, hsz = r * n;
  double* buf = (double*)malloc(sizeof(double) * (3 * wsz + 3 * hsz + 4 * r * r + r * n + 5 * m * r));
  st.w = buf; st.w_y = st.w + wsz; st.w_n = st.w_y + wsz;
  st.h = st.w_n + wsz; st.h_y = st.h + hsz; st.h_n = st.h_y + hsz;
  double* ws = st.h_n + hsz;
  memcpy(st.w, w0, sizeof(double) * wsz); memcpy(st.w_y, w0, sizeof(double) * wsz);
  memcpy(st.h, h0, sizeof(double) * hsz); memcpy(st.h_y, h0, sizeof(double) * hsz);
  st.schedule.beta = cfg->beta0; st.schedule.beta_bar = 1.0; st.schedule.beta_prev = cfg->beta0;
  st.schedule.gamma = cfg->gamma; st.schedule.gamma_bar = cfg->gamma_bar; st.schedule.eta = cfg->eta;
  st.restarted = 0;
  if (g_orc_threads > 1) rep_gram_rows(h0, r, n, ws);
  else orc_gram_rows(h0, r, n, ws);
  x_cross_xht(&X, h0, r, ws + r * r);
  st.err_prev = orc_fast_error(nx2, w0, ws + r * r, ws, m, r);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  enmf_gpu_iter rec;
  memset(&rec, 0, sizeof rec);
  for (uint64_t k = 1; k <= nsteps && rc == ENMF_OK; ++k) rc = step(&X, nx2, &st, cfg, r, k, &rec, ws);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  if (last_rel_err) *last_rel_err = rec.relative_error;
  free(buf);
  return rc;
}

/* run()'s prologue, `nskip` untimed step() calls, then `nsteps` timed ones: *seconds = the time
 * inside those nsteps (the reference arm of bench.py times the same iteration window as the GPU
 * arm); recs (nsteps entries) receive their records. */
int orc_time_window(const double* x, size_t m, size_t n, const double* w0, const double* h0, size_t r,
                    const enmf_gpu_config* cfg, size_t nskip, size_t nsteps, double* seconds, enmf_gpu_iter* recs) {
  int rc = orc_config_validate(cfg);
  if (rc) return rc;
  xmat X = {0, x, NULL, NULL, NULL, m, n, m * n};
  const double nx2 = orc_frob_norm_sq(x, m * n);
  ext_state st;
  const size_t wsz = m * r, hsz = r * n;
  double* buf = (double*)malloc(sizeof(double) * (3 * wsz + 3 * hsz + 4 * r * r + r * n + 5 * m * r));
  st.w = buf; st.w_y = st.w + wsz; st.w_n = st.w_y + wsz;
  st.h = st.w_n + wsz; st.h_y = st.h + hsz; st.h_n = st.h_y + hsz;
  double* ws = st.h_n + hsz;
  memcpy(st.w, w0, sizeof(double) * wsz); memcpy(st.w_y, w0, sizeof(double) * wsz);
  memcpy(st.h, h0, sizeof(double) * hsz); memcpy(st.h_y, h0, sizeof(double) * hsz);
  st.schedule.beta = cfg->beta0; st.schedule.beta_bar = 1.0; st.schedule.beta_prev = cfg->beta0;
  st.schedule.gamma = cfg->gamma; st.schedule.gamma_bar = cfg->gamma_bar; st.schedule.eta = cfg->eta;
  st.restarted = 0;
  if (g_orc_threads > 1) rep_gram_rows(h0, r, n, ws);
  else orc_gram_rows(h0, r, n, ws);
  x_cross_xht(&X, h0, r, ws + r * r);
  st.err_prev = orc_fast_error(nx2, w0, ws + r * r, ws, m, r);
  enmf_gpu_iter rec;
  memset(&rec, 0, sizeof rec);
  uint64_t k = 1;
  for (; k <= nskip && rc == ENMF_OK; ++k) rc = step(&X, nx2, &st, cfg, r, k, &rec, ws);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (size_t i = 0; i < nsteps && rc == ENMF_OK; ++i, ++k) {
    rc = step(&X, nx2, &st, cfg, r, k, &rec, ws);
    if (recs) recs[i] = rec;
  }
  clock_gettime(CLOCK_MONOTONIC, &t1);
  *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  free(buf);
  return rc;
}

int orc_run_dense(const double* x, size_t m, size_t n, const double* w0, const double* h0, size_t r,
                  const enmf_gpu_config* cfg, enmf_gpu_iter* iters, size_t iters_cap,
                  size_t* n_iters, double* w_out, double* h_out, double* norm_x) {
  xmat X = {0, x, NULL, NULL, NULL, m, n, m * n};
  return run_impl(&X, w0, h0, r, cfg, iters, iters_cap, n_iters, w_out, h_out, norm_x);
}

int orc_run_csr(const uint64_t* off, const uint64_t* cidx, const double* vals, size_t m, size_t n,
                size_t nnz, const double* w0, const double* h0, size_t r,
                const enmf_gpu_config* cfg, enmf_gpu_iter* iters, size_t iters_cap,
                size_t* n_iters, double* w_out, double* h_out, double* norm_x) {
  xmat X = {1, NULL, off, cidx, vals, m, n, nnz};
  return run_impl(&X, w0, h0, r, cfg, iters, iters_cap, n_iters, w_out, h_out, norm_x);
}

/* ----------------------------------------------------------------- data.hpp */
/* lowrank_factors + gen_lowrank, data.hpp:62-80 */
void orc_gen_lowrank(size_t m, size_t n, size_t r, uint64_t seed, double* x) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  double* w = (double*)malloc(sizeof(double) * m * r);
  double* h = (double*)malloc(sizeof(double) * r * n);
  fill_uniform(w, m * r, &g);
  fill_uniform(h, r * n, &g);
  multiply(w, h, m, r, n, x);
  free(w); free(h);
}

/* gen_fullrank, data.hpp:84-86 */
void orc_gen_fullrank(size_t m, size_t n, uint64_t seed, double* x) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  fill_uniform(x, m * n, &g);
}

/* random_init, data.hpp:90-97 */
void orc_random_init(size_t m, size_t n, size_t r, uint64_t seed, double* w, double* h) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  fill_uniform(w, m * r, &g);
  fill_uniform(h, r * n, &g);
}

/* ------------------------------------------- BASELINE.json config generators
 * NOT in the reference (data.hpp only has gen_lowrank / gen_fullrank).  They
 * realise the BASELINE.json config descriptions; every draw comes from one
 * mt19937_64 stream seeded with `seed`, in the order documented here, and the
 * normal variates use Box–Muller on two uniform_unit draws (cosine branch only). */
static double normal01(orc_mt64* g) {
  const double u1 = orc_uniform_unit(g), u2 = orc_uniform_unit(g);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
}

/* which = 2: X = W0·H0 + |N(0, 0.01²)|, W0 70% zeros (draw z, v per entry:
 *            W0 = z < 0.7 ? 0 : v), H0 uniform; X /= max(X)        (config 2)
 * which = 3: X = max(0, W0·H0 + N(0, (0.05·mean(W0·H0))²))           (config 3)
 * which = 5: X = W0·H0 + |N(0, 0.01²)|, W0/H0 uniform                (config 5)
 * Order: W0 row-major, H0 row-major, then one normal per X entry row-major. */
int orc_gen_config(int which, size_t m, size_t n, size_t r, uint64_t seed, double* x) {
  if (which != 2 && which != 3 && which != 5) { set_err("gen_config: which must be 2, 3 or 5"); return ENMF_INVALID_ARGUMENT; }
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  double* w = (double*)calloc(m * r, sizeof(double));
  double* h = (double*)calloc(r * n, sizeof(double));
  if (which == 2) {
    for (size_t i = 0; i < m * r; ++i) {
      const double z = orc_uniform_unit(&g), v = orc_uniform_unit(&g);
      w[i] = z < 0.7 ? 0.0 : v;
    }
  } else {
    fill_uniform(w, m * r, &g);
  }
  fill_uniform(h, r * n, &g);
  multiply(w, h, m, r, n, x);
  free(w); free(h);
  if (which == 3) {
    double s = 0.0;
    for (size_t i = 0; i < m * n; ++i) s += x[i];
    const double sigma = 0.05 * (s / (double)(m * n));
    for (size_t i = 0; i < m * n; ++i) {
      const double v = x[i] + sigma * normal01(&g);
      x[i] = v > 0.0 ? v : 0.0;
    }
  } else {
    for (size_t i = 0; i < m * n; ++i) x[i] += 0.01 * fabs(normal01(&g));
    if (which == 2) {
      double mx = 0.0;
      for (size_t i = 0; i < m * n; ++i) mx = x[i] > mx ? x[i] : mx;
      for (size_t i = 0; i < m * n; ++i) x[i] /= mx;
    }
  }
  return ENMF_OK;
}

/* Config 4: document-shaped CSR, rows = terms (m), cols = docs (n).
 * Per doc j (in order): L = max(1, round(exp(5 + N(0,1)))); L term ids drawn
 * Zipf(s) over ranks 1..m (inverse CDF by binary search, rank q -> term q-1).
 * Values tf·log(n/df) (zero weights dropped), then each column L2-normalised.
 * Arrays are malloc'ed; free with orc_free. */
static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}
int orc_gen_docs(size_t m, size_t n, double zipf_s, uint64_t seed, uint64_t** off_out,
                 uint64_t** cidx_out, double** vals_out, size_t* nnz_out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  double* cw = (double*)malloc(sizeof(double) * m);
  double tot = 0.0;
  for (size_t q = 0; q < m; ++q) { tot += pow((double)(q + 1), -zipf_s); cw[q] = tot; }
  size_t cap = 1 << 20, cnt = 0;
  uint32_t* tr = (uint32_t*)malloc(sizeof(uint32_t) * cap);   /* term */
  uint32_t* dc = (uint32_t*)malloc(sizeof(uint32_t) * cap);   /* doc */
  double* tf = (double*)malloc(sizeof(double) * cap);
  uint32_t* buf = NULL; size_t bufcap = 0;
  for (size_t j = 0; j < n; ++j) {
    double ll = exp(5.0 + normal01(&g));
    size_t L = (size_t)llround(ll);
    if (L < 1) L = 1;
    if (L > bufcap) { bufcap = L * 2; buf = (uint32_t*)realloc(buf, sizeof(uint32_t) * bufcap); }
    for (size_t t = 0; t < L; ++t) {
      const double u = orc_uniform_unit(&g) * tot;
      size_t lo = 0, hi = m - 1;
      while (lo < hi) { size_t mid = (lo + hi) / 2; if (cw[mid] > u) hi = mid; else lo = mid + 1; }
      buf[t] = (uint32_t)lo;
    }
    qsort(buf, L, sizeof(uint32_t), cmp_u32);
    for (size_t t = 0; t < L;) {
      size_t e = t;
      while (e < L && buf[e] == buf[t]) ++e;
      if (cnt == cap) {
        cap *= 2;
        tr = (uint32_t*)realloc(tr, sizeof(uint32_t) * cap);
        dc = (uint32_t*)realloc(dc, sizeof(uint32_t) * cap);
        tf = (double*)realloc(tf, sizeof(double) * cap);
      }
      tr[cnt] = buf[t]; dc[cnt] = (uint32_t)j; tf[cnt] = (double)(e - t); ++cnt;
      t = e;
    }
  }
  free(buf);
  uint64_t* df = (uint64_t*)calloc(m, sizeof(uint64_t));
  for (size_t p = 0; p < cnt; ++p) df[tr[p]]++;
  double* colsq = (double*)calloc(n, sizeof(double));
  for (size_t p = 0; p < cnt; ++p) {
    tf[p] = tf[p] * log((double)n / (double)df[tr[p]]);
    colsq[dc[p]] += tf[p] * tf[p];
  }
  uint64_t* off = (uint64_t*)calloc(m + 1, sizeof(uint64_t));
  size_t nnz = 0;
  for (size_t p = 0; p < cnt; ++p) if (tf[p] != 0.0) { off[tr[p] + 1]++; ++nnz; }
  for (size_t i = 0; i < m; ++i) off[i + 1] += off[i];
  uint64_t* cidx = (uint64_t*)malloc(sizeof(uint64_t) * (nnz ? nnz : 1));
  double* vals = (double*)malloc(sizeof(double) * (nnz ? nnz : 1));
  uint64_t* fillp = (uint64_t*)malloc(sizeof(uint64_t) * m);
  for (size_t i = 0; i < m; ++i) fillp[i] = off[i];
  /* entries are generated doc-major with ascending terms per doc, so scanning
   * them in order fills every CSR row with strictly increasing doc ids. */
  for (size_t p = 0; p < cnt; ++p) {
    if (tf[p] == 0.0) continue;
    const uint64_t q = fillp[tr[p]]++;
    cidx[q] = dc[p];
    vals[q] = tf[p] / sqrt(colsq[dc[p]]);
  }
  free(fillp); free(colsq); free(df); free(tr); free(dc); free(tf); free(cw);
  *off_out = off; *cidx_out = cidx; *vals_out = vals; *nnz_out = nnz;
  return ENMF_OK;
}

void orc_free(void* p) { free(p); }

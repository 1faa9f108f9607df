/*
 * enmf_oracle.h — CPU restatement of the reference enmf hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 path; it
 * is imported/linked only by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs.  The product (paper_1805_06604_b200,
 * libenmf_gpu.so) never calls it and has no CPU fallback.
 *
 * Every function restates one reference function with the same floating-point
 * operation order, so that built with -O2 -ffp-contract=off (separately rounded
 * multiply and add, as the reference's baseline x86-64 build) it is bitwise
 * identical to the reference.  Pinned against the reference itself compiled
 * from /root/reference (oracle/_ref, see oracle/Makefile) and against the
 * reference's known answers (tests/golden/, tests/test_oracle.py).
 */
#ifndef ENMF_ORACLE_H_
#define ENMF_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/enmf_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp ---- */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;   /* std::mt19937_64 */
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
uint64_t orc_mix64(uint64_t z);                                   /* rng.hpp:30-34 */
uint64_t orc_mix_seed(uint64_t base, uint64_t a, uint64_t b);     /* rng.hpp:38-44 */
double orc_uniform_unit(orc_mt64* g);                             /* rng.hpp:47-49 */

/* ---- data.hpp generators ---- */
/* gen_lowrank (data.hpp:76-80): x m×n */
void orc_gen_lowrank(size_t m, size_t n, size_t r, uint64_t seed, double* x);
/* gen_fullrank (data.hpp:84-86) */
void orc_gen_fullrank(size_t m, size_t n, uint64_t seed, double* x);
/* random_init (data.hpp:90-97): w m×r then h r×n from one stream */
void orc_random_init(size_t m, size_t n, size_t r, uint64_t seed, double* w, double* h);

/* ---- linalg.hpp ---- */
void orc_gram(const double* a, size_t m, size_t r, double* g);                 /* :49-64 */
void orc_gram_rows(const double* t, size_t r, size_t n, double* g);            /* gram(tᵀ) */
void orc_cross_wx(const double* w, const double* x, size_t m, size_t n, size_t r, double* out);   /* :67-83 */
void orc_cross_xht(const double* x, const double* h, size_t m, size_t n, size_t r, double* out);  /* :107-124 */
void orc_cross_wx_csr(const double* w, const uint64_t* off, const uint64_t* cidx, const double* v,
                      size_t m, size_t n, size_t r, double* out);                /* :86-104 */
void orc_cross_xht_csr(const uint64_t* off, const uint64_t* cidx, const double* v, const double* h,
                       size_t m, size_t n, size_t r, double* out);               /* :127-146 */
double orc_frob_norm_sq(const double* x, size_t count);                        /* :160-171 */
double orc_fast_error(double norm_x_sq, const double* w, const double* xht, const double* hht,
                      size_t m, size_t r);                                      /* engine.hpp:121-136 */

/* ---- nnls.hpp ---- */
/* hals_solve (nnls.hpp:154-176): returns ENMF_OK / ENMF_DEGENERATE_COLUMN. */
int orc_hals_solve(const double* gram, const double* cross, const double* h0, size_t r, size_t n,
                   uint64_t max_sweeps, double stall_fraction, double* h, int32_t* sweeps);
/* active_set_solve (nnls.hpp:259-406): returns ENMF_OK / ENMF_NO_CONVERGENCE. */
int orc_active_set_solve(const double* gram, const double* cross, const double* h0, size_t r,
                         size_t n, double* h, int32_t* rounds);
/* the same on a shard of the columns, with the whole problem's max|cross| and column count */
int orc_active_set_solve_shard(const double* gram, const double* cross, const double* h0, size_t r, size_t n,
                               double cmax_all, size_t n_all, double* h, int32_t* rounds, uint64_t* exch_out);
void orc_uniform_stream(uint64_t seed, size_t count, double* out);
uint64_t orc_derive_max_sweeps(double setup_flops, double sweep_flops, double ratio);  /* :79-87 */

/* ---- engine.hpp ---- */
enmf_gpu_beta_schedule orc_update_beta(enmf_gpu_beta_schedule s, int error_decreased); /* :88-99 */
int orc_config_validate(const enmf_gpu_config* cfg);                                  /* :175-199 */

/* run<DenseMatrix> (engine.hpp:447-521) with TimingMode::none semantics for
 * elapsed (always 0).  Same signature as enmf_gpu_run_dense minus the ctx. */
int orc_run_dense(const double* x, size_t m, size_t n, const double* w0, const double* h0, size_t r,
                  const enmf_gpu_config* cfg, enmf_gpu_iter* iters, size_t iters_cap,
                  size_t* n_iters, double* w_out, double* h_out, double* norm_x);
int orc_run_csr(const uint64_t* off, const uint64_t* cidx, const double* vals, size_t m, size_t n,
                size_t nnz, const double* w0, const double* h0, size_t r,
                const enmf_gpu_config* cfg, enmf_gpu_iter* iters, size_t iters_cap,
                size_t* n_iters, double* w_out, double* h_out, double* norm_x);

/* run()'s prologue + nsteps step() calls; *seconds = time inside step() only. */
int orc_time_steps(const double* x, size_t m, size_t n, const double* w0, const double* h0, size_t r,
                   const enmf_gpu_config* cfg, size_t nsteps, double* seconds, double* last_rel_err);

/* prologue + nskip untimed steps + nsteps timed steps (their records into recs) */
int orc_time_window(const double* x, size_t m, size_t n, const double* w0, const double* h0, size_t r,
                    const enmf_gpu_config* cfg, size_t nskip, size_t nsteps, double* seconds, enmf_gpu_iter* recs);

/* BASELINE.json config generators (new; not in the reference) */
int orc_gen_config(int which, size_t m, size_t n, size_t r, uint64_t seed, double* x);
int orc_gen_docs(size_t m, size_t n, double zipf_s, uint64_t seed, uint64_t** off, uint64_t** cidx,
                 double** vals, size_t* nnz);
void orc_free(void* p);

/* ---- replica.c: bit-exact multi-threaded execution of the dense path ----
 * n > 1 routes cross_wx, cross_xht, gram and hals_solve of orc_run_dense /
 * orc_time_steps through OpenMP kernels that keep every element's reference
 * summation order (bitwise identical results); 1 = the plain port. */
void orc_set_threads(int n);
int orc_get_threads(void);
/* C5 data (X = W0·H0 + 0.01·|N(0,1)|) on T×T tiles with per-tile streams (replica.c). */
int orc_gen_tiled(size_t m, size_t n, size_t r, uint64_t seed, size_t T, double* x);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif

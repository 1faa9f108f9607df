/*
 * enmf_gpu.h — C-ABI of the B200-native extrapolated-NMF hot path.
 *
 * This is the drop-in boundary for the per-outer-iteration path of the
 * reference library `enmf` (header-only C++20, /root/reference/proj/include/enmf).
 * The reference has no FFI layer: its boundary is the template API
 *
 *   RunRecord enmf::run(const MatrixX& x, const DenseMatrix& w0, const DenseMatrix& h0,
 *                       const SolverConfig& cfg, TimingMode timing)       engine.hpp:447-449
 *   IterationRecord enmf::step(...)                                      engine.hpp:309-311
 *
 * Every entry point below replaces one of those (or one of the public kernels
 * the reference's own tests call: gram / cross_wx / cross_xht / hals_solve /
 * active_set_solve / fast_error / update_beta).  Plain pointers and sizes only;
 * all matrices are row-major FP64 exactly as `enmf::DenseMatrix` stores them
 * (matrix.hpp:65-66: element (i,j) at v[i*cols+j]); CSR uses 64-bit offsets and
 * column indices like `enmf::SparseMatrix` (matrix.hpp:255-257).
 *
 * Errors: the reference throws C++ exceptions; here every call returns one of
 * the ENMF_* codes below and the message is available from enmf_gpu_last_error()
 * (thread-local).  include/enmf_gpu.hpp maps the codes back onto the reference's
 * exception types.
 *
 * Thread safety: one enmf_gpu_ctx per calling thread.  Distinct contexts may be
 * used concurrently (the reference's run_suite runs independent run() calls on a
 * thread pool, bench.hpp:273-292).
 */
#ifndef ENMF_GPU_H_
#define ENMF_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes (reference exception → code). */
enum {
  ENMF_OK = 0,
  ENMF_INVALID_ARGUMENT = 1,   /* std::invalid_argument          engine.hpp:175-199,450-459 */
  ENMF_NON_FINITE = 2,         /* enmf::NonFiniteIterate          engine.hpp:51-54 */
  ENMF_NO_CONVERGENCE = 3,     /* enmf::NoConvergence             nnls.hpp:65-68, engine.hpp:290-292 */
  ENMF_DEGENERATE_COLUMN = 4,  /* enmf::DegenerateColumn          nnls.hpp:54-63 */
  ENMF_CUDA_ERROR = 5,         /* device / driver failure (no reference analogue) */
  ENMF_CACHE_STALE = 6,        /* enmf::CacheStale                engine.hpp:41-44 */
  ENMF_PARSE_ERROR = 7,        /* enmf::ParseError (+ line)       data.hpp:34-43 */
  ENMF_UNSUPPORTED_FORMAT = 8, /* enmf::UnsupportedFormat         data.hpp:45-48 */
  ENMF_IO_ERROR = 9,           /* enmf::IoError                   data.hpp:50-53 */
  ENMF_ZERO_DIRECTION = 10     /* enmf::ZeroDirection             engine.hpp:46-49 */
};

/* enmf::InnerSolver (engine.hpp:56) */
enum { ENMF_INNER_EXACT = 0, ENMF_INNER_HALS = 1 };
/* enmf::TimingMode (engine.hpp:58) */
enum { ENMF_TIMING_WALL = 0, ENMF_TIMING_NONE = 1 };
/* Arithmetic of the device path. FP64 is the parity path. */
enum {
  ENMF_PRECISION_FP64 = 0,        /* DMMA tensor-core GEMMs, FMA sweeps: the product path */
  ENMF_PRECISION_TF32 = 1,        /* variant: W_yᵀX and X·Tᵀ on TF32 tensor cores (X held in FP32), rest FP64 */
  ENMF_PRECISION_FP64_EXACT = 2   /* bitwise-faithful debug path: reference summation order, no FMA */
};

/* 1:1 with enmf::SolverConfig (engine.hpp:149-173).  `inner_max_sweeps` = 0
 * means "std::nullopt" (derive from the setup/sweep cost ratio). */
typedef struct enmf_gpu_config {
  int32_t inner_h;               /* ENMF_INNER_* */
  int32_t inner_w;               /* ENMF_INNER_* */
  int32_t hp;                    /* 1 | 2 | 3 */
  int32_t extrapolation_enabled; /* bool */
  double beta0;
  double gamma;
  double gamma_bar;
  double eta;
  uint64_t max_outer_iterations;
  double max_seconds;            /* +inf = no budget */
  int32_t literal_hp1_order;     /* bool */
  int32_t timing;                /* ENMF_TIMING_* */
  double inner_sweep_ratio;
  double inner_stall_fraction;
  uint64_t inner_max_sweeps;     /* 0 = derive */
  uint64_t reinit_seed;
  int32_t precision;             /* ENMF_PRECISION_* */
  int32_t reserved;
} enmf_gpu_config;

/* enmf::IterationRecord (engine.hpp:216-223) plus per-iteration
 * instrumentation the reference does not record (used by parity tests). */
typedef struct enmf_gpu_iter {
  uint64_t iteration;
  double elapsed_seconds;
  double error;
  double relative_error;
  double beta;
  int32_t restarted;
  int32_t inner_h_count;   /* HALS sweeps (or BPP rounds) of the H update */
  int32_t inner_w_count;   /* HALS sweeps (or BPP rounds) of the W update */
  int32_t reinit_events;   /* bit0: W_y columns redrawn, bit1: target rows redrawn */
} enmf_gpu_iter;

/* enmf::BetaSchedule (engine.hpp:63-70) */
typedef struct enmf_gpu_beta_schedule {
  double beta, beta_bar, beta_prev, gamma, gamma_bar, eta;
} enmf_gpu_beta_schedule;

typedef struct enmf_gpu_ctx enmf_gpu_ctx;

/* Fills `cfg` with the defaults of enmf::SolverConfig (engine.hpp:149-173). */
void enmf_gpu_config_default(enmf_gpu_config* cfg);
/* Named presets of enmf::detail::algorithm_config (bench.hpp:108-135):
 * "anls", "e-anls-hp1", "e-anls-hp3", "ahals", "e-ahals-hp1", "e-ahals-hp3". */
int enmf_gpu_config_preset(enmf_gpu_config* cfg, const char* name);
/* SolverConfig::validate (engine.hpp:175-199). */
int enmf_gpu_config_validate(const enmf_gpu_config* cfg);
/* update_beta (engine.hpp:88-99) — host scalar logic, identical on device. */
enmf_gpu_beta_schedule enmf_gpu_update_beta(enmf_gpu_beta_schedule s, int error_decreased);

/* Context: owns the CUDA stream, device buffers and captured graphs.
 * device < 0 selects the current device. */
int enmf_gpu_create(enmf_gpu_ctx** out, int device);
void enmf_gpu_destroy(enmf_gpu_ctx* ctx);
const char* enmf_gpu_last_error(void);
/* Line of the last ENMF_PARSE_ERROR (enmf::ParseError::line(), data.hpp:39); 0 = none. */
size_t enmf_gpu_last_error_line(void);
/* Number of device kernels this context has launched since creation. */
uint64_t enmf_gpu_kernel_launches(const enmf_gpu_ctx* ctx);

/* ---- drop-in for enmf::run<DenseMatrix> (engine.hpp:447-521) ----------------
 * x: m×n, w0: m×r, h0: r×n (host, row-major).  iters receives entries 0..K
 * (entry 0 = initial pair), at most iters_cap of them; *n_iters gets the count.
 * w_out (m×r) / h_out (r×n) receive RunRecord::factors; *norm_x = ‖X‖_F. */
int enmf_gpu_run_dense(enmf_gpu_ctx* ctx, const double* x, size_t m, size_t n,
                       const double* w0, const double* h0, size_t r,
                       const enmf_gpu_config* cfg, enmf_gpu_iter* iters, size_t iters_cap,
                       size_t* n_iters, double* w_out, double* h_out, double* norm_x);

/* ---- drop-in for enmf::run<SparseMatrix> (engine.hpp:447-521 with the CSR
 * kernels linalg.hpp:86-104,127-146,167-171).  offsets: m+1, col_idx/vals: nnz. */
int enmf_gpu_run_csr(enmf_gpu_ctx* ctx, const uint64_t* offsets, const uint64_t* col_idx,
                     const double* vals, size_t m, size_t n, size_t nnz,
                     const double* w0, const double* h0, size_t r,
                     const enmf_gpu_config* cfg, enmf_gpu_iter* iters, size_t iters_cap,
                     size_t* n_iters, double* w_out, double* h_out, double* norm_x);

/* ---- packed many-small-runs backend (batch.cuh; the paper protocol's run grid,
 * bench.hpp:233-294): `count` independent dense runs of one shape and config, one CTA per
 * run, one launch for the whole batch.  x: count × m × n, w0: count × m × r, h0: count × r × n
 * (row-major, packed); outputs per run: iters_cap records (iters + b·iters_cap), n_iters[b],
 * status[b] (ENMF_* of that run), w_out, h_out, norm_x.  FP64 product mode, HALS or BPP (r <= 32,
 * max(m, n)·⌈r⌉₈ <= 9216, no wall budget): enmf_gpu_batch_eligible says whether a config fits. */
int enmf_gpu_batch_eligible(size_t m, size_t n, size_t r, const enmf_gpu_config* cfg);
int enmf_gpu_run_batch_dense(enmf_gpu_ctx* ctx, size_t count, const double* x, size_t m, size_t n,
                             const double* w0, const double* h0, size_t r, const enmf_gpu_config* cfg,
                             enmf_gpu_iter* iters, size_t iters_cap, int32_t* n_iters, int32_t* status,
                             double* w_out, double* h_out, double* norm_x);

/* Upload a CSR X (validated as SparseMatrix::validate, matrix.hpp:226-251) for
 * enmf_gpu_solve / enmf_gpu_begin; keeps a CSC copy on the device for W_yᵀX. */
int enmf_gpu_load_csr(enmf_gpu_ctx* ctx, const uint64_t* offsets, const uint64_t* col_idx,
                      const double* vals, size_t m, size_t n, size_t nnz);

/* ---- resident-data API (bench / repeated solves on one X) -------------------
 * Upload X once (from host or from a device pointer), then solve from device
 * or host factors.  *_device pointers are CUDA device pointers. */
int enmf_gpu_load_dense(enmf_gpu_ctx* ctx, const double* x, size_t m, size_t n, int x_on_device);
int enmf_gpu_solve(enmf_gpu_ctx* ctx, const double* w0, const double* h0, size_t r,
                   int factors_on_device, const enmf_gpu_config* cfg, enmf_gpu_iter* iters,
                   size_t iters_cap, size_t* n_iters, double* w_out, double* h_out,
                   double* norm_x);

/* ---- run session: enmf::run split into its phases (bench / step-wise drivers) --
 * begin = run()'s prologue (validation, upload, ||X||^2, e(0), capture of one
 * outer iteration as a CUDA graph); step = enqueue `count` more outer
 * iterations (engine.hpp:309-440), asynchronous on the context stream; sync =
 * wait and read records 0..k (returns the error code of a failed iteration);
 * end = RunRecord::factors (engine.hpp:518-520) and close.  X must already be
 * loaded (enmf_gpu_load_dense).  At most cfg->max_outer_iterations steps. */
int enmf_gpu_begin(enmf_gpu_ctx* ctx, const double* w0, const double* h0, size_t r,
                   int factors_on_device, const enmf_gpu_config* cfg);
int enmf_gpu_step(enmf_gpu_ctx* ctx, uint64_t count);
/* One outer iteration launched kernel by kernel with CUDA events between the
 * phases; phase_ms[0..10] = {gram(W_y)+reinit, W_yᵀX, H update, H extrapolation,
 * gram(T)+reinit, X·Tᵀ, W update, error products, decide+finalize,
 * H sweeps, W sweeps}.  Advances the run like enmf_gpu_step(ctx, 1). */
int enmf_gpu_step_profiled(enmf_gpu_ctx* ctx, double* phase_ms, size_t cap);
int enmf_gpu_sync(enmf_gpu_ctx* ctx, enmf_gpu_iter* iters, size_t iters_cap, size_t* n_iters);
int enmf_gpu_end(enmf_gpu_ctx* ctx, double* w_out, double* h_out, double* norm_x);
/* The context's CUDA stream (cudaStream_t) — for event timing by the caller. */
void* enmf_gpu_stream(enmf_gpu_ctx* ctx);
/* Digit levels S of the INT8-digit cross products for the loaded X (S(S+1)/2 int8 digit
 * GEMMs per product; 0 = that product runs on the FP64 DMMA GEMM or X is not loaded):
 * levels[0] for W_yᵀX, levels[1] for X·Tᵀ.  Reporting only (bench roofline). */
int enmf_gpu_digit_levels(const enmf_gpu_ctx* ctx, int32_t* levels);

/* ---- multi-GPU: one problem sharded over `world` GPUs ----------
 * One process per GPU.  Rank p owns rows [row0, row0+mp) of W and X (row block,
 * for X·Tᵀ) and columns [col0, col0+np) of H and X (column block, for W_yᵀX).
 * Setup: (1) every rank: enmf_gpu_dist_alloc -> a cudaIpcMemHandle_t (64 bytes)
 * of its shared block; (2) the caller all-gathers the handles (any host
 * channel, e.g. torch.distributed); (3) every rank: enmf_gpu_dist_init with the
 * world × 64-byte handle array; (4) a host barrier; (5) enmf_gpu_load_dense_sharded.
 * Runs then use enmf_gpu_begin/step/sync/end (or enmf_gpu_solve) with this
 * rank's factor shards: w0 = W0[row0:row0+mp, :] (mp × r), h0 = H0[:, col0:col0+np]
 * (r × np); outputs are the same shards.  Records are identical on all ranks. */
void enmf_gpu_dist_shard(size_t m, size_t n, int rank, int world, size_t* row0, size_t* mp,
                         size_t* col0, size_t* np);
int enmf_gpu_dist_alloc(enmf_gpu_ctx* ctx, int rank, int world, size_t m, size_t n, size_t r,
                        void* ipc_handle_out);
int enmf_gpu_dist_init(enmf_gpu_ctx* ctx, const void* ipc_handles);
int enmf_gpu_load_dense_sharded(enmf_gpu_ctx* ctx, const double* x_cols, const double* x_rows,
                                int on_device);
int enmf_gpu_dist_finalize(enmf_gpu_ctx* ctx);
/* Self-test of the cross-rank exchange primitives (epoch flags, double-buffered mailbox slots,
 * rank-ordered sums, shard all-gather + barrier) with `world` ranks on THIS GPU: one cooperative
 * launch, block p = rank p, `epochs` rounds of every exchange the sharded engine uses.  in:
 * [world][count] contributions; red: [world][epochs][count] all-reduced values; sc:
 * [world][epochs][3] = (gain sum, flag OR, max); rep_w / rep_t: [world][r*full] each rank's
 * replicas after the last round.  (No reference analogue: the reference is single-process.) */
int enmf_gpu_dist_selftest(enmf_gpu_ctx* ctx, int world, int count, int epochs, int r, size_t full,
                           const double* in, double* red, double* sc, double* rep_w, double* rep_t);

/* hals_solve (nnls.hpp:154-176) of an r x n problem sharded by columns over `world` ranks that all
 * run on THIS GPU in one cooperative launch (64 < r <= 128): the sharded engine's sweep path — the
 * synchronous grid decision with the per-sweep cross-rank gain exchange — with every rank
 * co-resident.  h: r x n result; sweeps: world entries, identical on every rank. */
int enmf_gpu_hals_solve_vranks(enmf_gpu_ctx* ctx, const double* gram, const double* cross, const double* h0,
                               size_t r, size_t n, int world, uint64_t max_sweeps, double stall_fraction,
                               double* h, int32_t* sweeps);

/* ---- public kernels the reference's tests call (host pointers) --------------
 * They run in the context's kernel precision (default ENMF_PRECISION_FP64). */
int enmf_gpu_set_precision(enmf_gpu_ctx* ctx, int precision);
/* gram (linalg.hpp:49-64): a m×r → g r×r, bitwise symmetric. */
int enmf_gpu_gram(enmf_gpu_ctx* ctx, const double* a, size_t m, size_t r, double* g);
/* cross_wx (linalg.hpp:67-83): w m×r, x m×n → out r×n. */
int enmf_gpu_cross_wx(enmf_gpu_ctx* ctx, const double* w, const double* x, size_t m, size_t n,
                      size_t r, double* out);
/* cross_xht (linalg.hpp:107-124): x m×n, h r×n → out m×r. */
int enmf_gpu_cross_xht(enmf_gpu_ctx* ctx, const double* x, const double* h, size_t m, size_t n,
                       size_t r, double* out);
/* frob_norm_sq (linalg.hpp:160-171), compensated. */
int enmf_gpu_frob_norm_sq(enmf_gpu_ctx* ctx, const double* x, size_t count, double* out);
/* fast_error (engine.hpp:121-136): w m×r, xht m×r, hht r×r. */
int enmf_gpu_fast_error(enmf_gpu_ctx* ctx, double norm_x_sq, const double* w, const double* xht,
                        const double* hht, size_t m, size_t r, double* err);
/* hals_solve (nnls.hpp:154-176) with InnerLoopPolicy{max_sweeps, stall_fraction}:
 * gram r×r, cross r×n, h0 r×n → h r×n; *sweeps = sweeps performed. */
int enmf_gpu_hals_solve(enmf_gpu_ctx* ctx, const double* gram, const double* cross,
                        const double* h0, size_t r, size_t n, uint64_t max_sweeps,
                        double stall_fraction, double* h, int32_t* sweeps);
/* active_set_solve (nnls.hpp:259-406): gram r×r, cross r×n, h0 r×n → h r×n;
 * *rounds = max exchange rounds over the columns. */
int enmf_gpu_active_set_solve(enmf_gpu_ctx* ctx, const double* gram, const double* cross,
                              const double* h0, size_t r, size_t n, double* h, int32_t* rounds);


/* optimal_beta_linesearch (engine.hpp:522-540), the diagnostic the reference's tests use:
 *   beta* = <X − W_n·H_y, (W_n − W)·H_y> / ||(W_n − W)·H_y||²
 * with W_n, W m×r and H_y r×n row-major host arrays; X dense (m×n) or CSR.  Returns
 * ENMF_ZERO_DIRECTION when ||(W_n − W)·H_y||² ≤ 1e-30·||X||² (ZeroDirection). */
int enmf_gpu_optimal_beta_linesearch(enmf_gpu_ctx* ctx, const double* x, size_t m, size_t n, const double* w_n,
                                     const double* w, const double* h_y, size_t r, double* beta);
int enmf_gpu_optimal_beta_linesearch_csr(enmf_gpu_ctx* ctx, const uint64_t* offsets, const uint64_t* col_idx,
                                         const double* vals, size_t m, size_t n, size_t nnz, const double* w_n,
                                         const double* w, const double* h_y, size_t r, double* beta);

/* ------------------------------------------------------------------------------------
 * Data formats and generators (host side, csrc/io.cpp): the reference's enmf/data.hpp.
 * Readers return a library-owned matrix; read its arrays, then enmf_io_matrix_free().
 * Sparse results are CSR exactly as SparseMatrix::from_triplets builds them
 * (matrix.hpp:168-195: rows ascending, columns ascending within a row). */
typedef struct enmf_io_matrix enmf_io_matrix;

/* read_matrix_market (data.hpp:159-240): coordinate real|integer general, 1-based. */
int enmf_io_read_matrix_market(const char* path, enmf_io_matrix** out);
/* read_dense_csv (data.hpp:262-295): headerless, comma separated, CRLF accepted. */
int enmf_io_read_dense_csv(const char* path, enmf_io_matrix** out);
void enmf_io_matrix_shape(const enmf_io_matrix* a, size_t* rows, size_t* cols, size_t* nnz, int* is_sparse);
const uint64_t* enmf_io_matrix_offsets(const enmf_io_matrix* a);      /* rows+1, sparse only */
const uint64_t* enmf_io_matrix_col_indices(const enmf_io_matrix* a);  /* nnz, sparse only */
const double* enmf_io_matrix_values(const enmf_io_matrix* a);         /* nnz, or rows*cols row-major */
void enmf_io_matrix_free(enmf_io_matrix* a);

/* write_matrix_market (data.hpp:242-257) / write_dense_csv (data.hpp:297-309) /
 * write_run_csv (data.hpp:316-326; E = relative_error - e_min). */
int enmf_io_write_matrix_market(const char* path, const uint64_t* offsets, const uint64_t* col_idx,
                                const double* vals, size_t rows, size_t cols);
int enmf_io_write_dense_csv(const char* path, const double* x, size_t rows, size_t cols);
int enmf_io_write_run_csv(const char* path, const enmf_gpu_iter* iters, size_t n, double e_min);
/* format_double (data.hpp:101-105): shortest round-trip form; returns its length and
 * writes at most cap-1 characters plus a terminator. */
size_t enmf_io_format_double(double v, char* buf, size_t cap);

/* Generators (data.hpp:58-97, rng.hpp:30-57): one std::mt19937_64 stream each,
 * uniform [0,1) = (g() >> 11) * 2^-53, row-major fill. */
uint64_t enmf_mix_seed(uint64_t base, uint64_t a, uint64_t b);
int enmf_uniform_matrix(size_t rows, size_t cols, uint64_t seed, double* out);
int enmf_random_init(size_t m, size_t n, size_t r, uint64_t seed, double* w, double* h);
int enmf_lowrank_factors(size_t m, size_t n, size_t r, uint64_t seed, double* w, double* h);
int enmf_gen_lowrank(size_t m, size_t n, size_t r, uint64_t seed, double* x);   /* X = W·H */
int enmf_gen_fullrank(size_t m, size_t n, uint64_t seed, double* x);
/* BASELINE configs[4] data on T×T tiles with per-tile streams (T = 0: 4096): the block rows
 * [row0, row0+rows) × cols [col0, col0+cols) of X = W0·H0 + 0.01·|N(0,1)| (multi-threaded;
 * identical bits for any thread count or blocking). */
int enmf_gen_tiled(size_t m, size_t n, size_t r, uint64_t seed, size_t T, size_t row0, size_t rows, size_t col0,
                   size_t cols, double* x);

#ifdef __cplusplus
}
#endif

#endif /* ENMF_GPU_H_ */

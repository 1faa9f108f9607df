// enmf_gpu.hpp — header-only C++ shim: the reference's run() API on the B200 path.
//
// A caller of the reference (`enmf::run(x, w0, h0, cfg, timing)`,
// /root/reference/proj/include/enmf/engine.hpp:447-449) switches to the GPU by
// namespace:  enmf::run(...)  ->  enmf::gpu::run(...).  Same argument types
// (enmf::DenseMatrix / enmf::SparseMatrix / enmf::SolverConfig / TimingMode),
// same return type (enmf::RunRecord) and the same exception types
// (std::invalid_argument, enmf::NonFiniteIterate, enmf::NoConvergence,
// enmf::DegenerateColumn, enmf::CacheStale).  Requires the reference's own
// headers on the include path (it reuses their types) and links against
// libenmf_gpu.so.  One context per thread (run_suite-safe, bench.hpp:273-292).
#pragma once

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <enmf/engine.hpp>
#include <enmf/matrix.hpp>
#include <enmf/nnls.hpp>

#include "enmf_gpu.h"

namespace enmf {
namespace gpu {

[[noreturn]] inline void raise(int code) {
  const std::string msg = enmf_gpu_last_error();
  switch (code) {
    case ENMF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case ENMF_NON_FINITE: throw NonFiniteIterate(msg);
    case ENMF_NO_CONVERGENCE: throw NoConvergence(msg);
    case ENMF_DEGENERATE_COLUMN: throw DegenerateColumn(0);
    case ENMF_CACHE_STALE: throw CacheStale(msg);
    default: throw std::runtime_error("enmf_gpu: " + msg);
  }
}

inline void check(int code) {
  if (code != ENMF_OK) raise(code);
}

/// Per-thread device context (stream + buffers), created on first use.
inline enmf_gpu_ctx* thread_context() {
  struct Holder {
    enmf_gpu_ctx* c = nullptr;
    ~Holder() { if (c) enmf_gpu_destroy(c); }
  };
  thread_local Holder h;
  if (!h.c) check(enmf_gpu_create(&h.c, -1));
  return h.c;
}

inline enmf_gpu_config to_c(const SolverConfig& s, TimingMode timing) {
  enmf_gpu_config c;
  enmf_gpu_config_default(&c);
  c.inner_h = s.inner_h == InnerSolver::exact ? ENMF_INNER_EXACT : ENMF_INNER_HALS;
  c.inner_w = s.inner_w == InnerSolver::exact ? ENMF_INNER_EXACT : ENMF_INNER_HALS;
  c.hp = s.hp;
  c.extrapolation_enabled = s.extrapolation_enabled ? 1 : 0;
  c.beta0 = s.beta0;
  c.gamma = s.gamma;
  c.gamma_bar = s.gamma_bar;
  c.eta = s.eta;
  c.max_outer_iterations = s.max_outer_iterations;
  c.max_seconds = s.max_seconds;
  c.literal_hp1_order = s.literal_hp1_order ? 1 : 0;
  c.timing = timing == TimingMode::wall ? ENMF_TIMING_WALL : ENMF_TIMING_NONE;
  c.inner_sweep_ratio = s.inner_sweep_ratio;
  c.inner_stall_fraction = s.inner_stall_fraction;
  c.inner_max_sweeps = s.inner_max_sweeps ? *s.inner_max_sweeps : 0;
  c.reinit_seed = s.reinit_seed;
  c.precision = ENMF_PRECISION_FP64;
  return c;
}

inline RunRecord to_record(const std::vector<enmf_gpu_iter>& it, size_t count, DenseMatrix w, DenseMatrix h,
                           double norm_x) {
  RunRecord out;
  for (size_t k = 0; k < count && k < it.size(); ++k) {
    IterationRecord r;
    r.iteration = it[k].iteration;
    r.elapsed_seconds = it[k].elapsed_seconds;
    r.error = it[k].error;
    r.relative_error = it[k].relative_error;
    r.beta = it[k].beta;
    r.restarted = it[k].restarted != 0;
    out.iterations.push_back(r);
  }
  out.factors.w = std::move(w);
  out.factors.h = std::move(h);
  out.norm_x = norm_x;
  return out;
}

/// enmf::run<DenseMatrix> on the GPU (engine.hpp:447-521).
inline RunRecord run(const DenseMatrix& x, const DenseMatrix& w0, const DenseMatrix& h0, const SolverConfig& cfg,
                     TimingMode timing = TimingMode::wall) {
  cfg.validate();
  if (w0.cols() != h0.rows()) throw std::invalid_argument("run: factor inner dimensions disagree");
  if (w0.rows() != x.rows() || h0.cols() != x.cols())
    throw std::invalid_argument("run: factor shapes do not match the data matrix");
  const enmf_gpu_config c = to_c(cfg, timing);
  const size_t cap = cfg.max_outer_iterations + 1;
  std::vector<enmf_gpu_iter> it(cap);
  size_t count = 0;
  DenseMatrix w(w0.rows(), w0.cols(), 0.0), h(h0.rows(), h0.cols(), 0.0);
  double norm_x = 0.0;
  check(enmf_gpu_run_dense(thread_context(), x.data(), x.rows(), x.cols(), w0.data(), h0.data(), w0.cols(), &c,
                           it.data(), cap, &count, w.data(), h.data(), &norm_x));
  return to_record(it, count, std::move(w), std::move(h), norm_x);
}

/// enmf::run<SparseMatrix> on the GPU (CSR layout of matrix.hpp:153-258).
inline RunRecord run(const SparseMatrix& x, const DenseMatrix& w0, const DenseMatrix& h0, const SolverConfig& cfg,
                     TimingMode timing = TimingMode::wall) {
  cfg.validate();
  if (w0.cols() != h0.rows()) throw std::invalid_argument("run: factor inner dimensions disagree");
  if (w0.rows() != x.rows() || h0.cols() != x.cols())
    throw std::invalid_argument("run: factor shapes do not match the data matrix");
  const enmf_gpu_config c = to_c(cfg, timing);
  const size_t cap = cfg.max_outer_iterations + 1;
  std::vector<enmf_gpu_iter> it(cap);
  size_t count = 0;
  DenseMatrix w(w0.rows(), w0.cols(), 0.0), h(h0.rows(), h0.cols(), 0.0);
  double norm_x = 0.0;
  static_assert(sizeof(std::size_t) == sizeof(uint64_t), "CSR indices are passed as 64-bit");
  check(enmf_gpu_run_csr(thread_context(), reinterpret_cast<const uint64_t*>(x.offsets().data()),
                         reinterpret_cast<const uint64_t*>(x.col_indices().data()), x.values().data(), x.rows(),
                         x.cols(), x.nnz(), w0.data(), h0.data(), w0.cols(), &c, it.data(), cap, &count, w.data(),
                         h.data(), &norm_x));
  return to_record(it, count, std::move(w), std::move(h), norm_x);
}

/// The reference's public kernels (linalg.hpp / nnls.hpp) on the GPU.
inline DenseMatrix gram(const DenseMatrix& a) {
  DenseMatrix g(a.cols(), a.cols(), 0.0);
  check(enmf_gpu_gram(thread_context(), a.data(), a.rows(), a.cols(), g.data()));
  return g;
}
inline DenseMatrix cross_wx(const DenseMatrix& w, const DenseMatrix& x) {
  if (w.rows() != x.rows()) throw std::invalid_argument("cross_wx: row count mismatch");
  DenseMatrix out(w.cols(), x.cols(), 0.0);
  check(enmf_gpu_cross_wx(thread_context(), w.data(), x.data(), x.rows(), x.cols(), w.cols(), out.data()));
  return out;
}
inline DenseMatrix cross_xht(const DenseMatrix& x, const DenseMatrix& h) {
  if (x.cols() != h.cols()) throw std::invalid_argument("cross_xht: column count mismatch");
  DenseMatrix out(x.rows(), h.rows(), 0.0);
  check(enmf_gpu_cross_xht(thread_context(), x.data(), h.data(), x.rows(), x.cols(), h.rows(), out.data()));
  return out;
}
inline DenseMatrix hals_solve(const NnlsProblem& p, const DenseMatrix& h0, const InnerLoopPolicy& policy) {
  policy.validate();
  DenseMatrix h(h0.rows(), h0.cols(), 0.0);
  int32_t sweeps = 0;
  check(enmf_gpu_hals_solve(thread_context(), p.gram.data(), p.cross.data(), h0.data(), h0.rows(), h0.cols(),
                            policy.max_sweeps, policy.stall_fraction, h.data(), &sweeps));
  return h;
}
inline DenseMatrix active_set_solve(const NnlsProblem& p, const DenseMatrix& h0) {
  DenseMatrix h(h0.rows(), h0.cols(), 0.0);
  int32_t rounds = 0;
  check(enmf_gpu_active_set_solve(thread_context(), p.gram.data(), p.cross.data(), h0.data(), h0.rows(),
                                  h0.cols(), h.data(), &rounds));
  return h;
}

}  // namespace gpu
}  // namespace enmf

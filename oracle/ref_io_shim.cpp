// ref_io_shim.cpp — C-ABI around the UNMODIFIED reference's data formats and suite harness.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against /root/reference/proj/include
// (read in place, never copied) and the nlohmann json.hpp bench.hpp includes, into
// oracle/_ref/libenmf_ref_io.so.  tests/golden/make_golden_io.py calls it to produce the
// fixtures that pin csrc/io.cpp (readers, writers, generators) and suite.py (run_suite,
// curves, ranking, emit) to the reference's own outputs.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <json.hpp>

#include <enmf/bench.hpp>
#include <enmf/data.hpp>

#include "../include/enmf_gpu.h"

namespace {
thread_local std::string g_err;
thread_local std::size_t g_line = 0;

template <class F>
int guard(F&& f) {
  g_line = 0;
  try {
    f();
    return ENMF_OK;
  } catch (const enmf::ParseError& e) { g_err = e.what(); g_line = e.line(); return ENMF_PARSE_ERROR;
  } catch (const enmf::UnsupportedFormat& e) { g_err = e.what(); return ENMF_UNSUPPORTED_FORMAT;
  } catch (const enmf::IoError& e) { g_err = e.what(); return ENMF_IO_ERROR;
  } catch (const std::invalid_argument& e) { g_err = e.what(); return ENMF_INVALID_ARGUMENT;
  } catch (const std::exception& e) { g_err = e.what(); return 99; }
}

template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}
}  // namespace

extern "C" {

const char* ref_io_last_error(void) { return g_err.c_str(); }
size_t ref_io_last_line(void) { return g_line; }
void ref_io_free(void* p) { std::free(p); }

int ref_io_read_mm(const char* path, size_t* rows, size_t* cols, size_t* nnz, uint64_t** off, uint64_t** idx,
                   double** val) {
  return guard([&] {
    const enmf::SparseMatrix s = enmf::read_matrix_market(path);
    *rows = s.rows();
    *cols = s.cols();
    *nnz = s.nnz();
    std::vector<uint64_t> o(s.offsets().begin(), s.offsets().end()), c(s.col_indices().begin(), s.col_indices().end());
    *off = dup(o);
    *idx = dup(c);
    *val = dup(s.values());
  });
}

int ref_io_read_csv(const char* path, size_t* rows, size_t* cols, double** val) {
  return guard([&] {
    const enmf::DenseMatrix d = enmf::read_dense_csv(path);
    *rows = d.rows();
    *cols = d.cols();
    *val = dup(std::vector<double>(d.data(), d.data() + d.size()));
  });
}

int ref_io_write_mm(const char* path, const uint64_t* off, const uint64_t* idx, const double* val, size_t rows,
                    size_t cols) {
  return guard([&] {
    const size_t nnz = off[rows];
    enmf::SparseMatrix s(rows, cols, std::vector<std::size_t>(off, off + rows + 1),
                         std::vector<std::size_t>(idx, idx + nnz), std::vector<double>(val, val + nnz));
    enmf::write_matrix_market(path, s);
  });
}

int ref_io_write_csv(const char* path, const double* x, size_t rows, size_t cols) {
  return guard([&] {
    enmf::write_dense_csv(path, enmf::DenseMatrix(rows, cols, std::vector<double>(x, x + rows * cols)));
  });
}

int ref_io_write_run_csv(const char* path, const enmf_gpu_iter* it, size_t n, double e_min) {
  return guard([&] {
    enmf::RunRecord rec;
    for (size_t k = 0; k < n; ++k) {
      enmf::IterationRecord r;
      r.iteration = it[k].iteration;
      r.elapsed_seconds = it[k].elapsed_seconds;
      r.error = it[k].error;
      r.relative_error = it[k].relative_error;
      r.beta = it[k].beta;
      r.restarted = it[k].restarted != 0;
      rec.iterations.push_back(r);
    }
    enmf::write_run_csv(path, rec, e_min);
  });
}

size_t ref_io_format_double(double v, char* buf, size_t cap) {
  const std::string s = enmf::format_double(v);
  if (cap) {
    const size_t k = std::min(s.size(), cap - 1);
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return s.size();
}

int ref_gen_fullrank(size_t m, size_t n, uint64_t seed, double* x) {
  return guard([&] {
    const enmf::DenseMatrix d = enmf::gen_fullrank(m, n, seed);
    std::memcpy(x, d.data(), sizeof(double) * d.size());
  });
}

int ref_lowrank_factors(size_t m, size_t n, size_t r, uint64_t seed, double* w, double* h) {
  return guard([&] {
    auto [a, b] = enmf::lowrank_factors(m, n, r, seed);
    std::memcpy(w, a.data(), sizeof(double) * a.size());
    std::memcpy(h, b.data(), sizeof(double) * b.size());
  });
}

// Runs enmf::run_suite on a JSON spec and enmf::emit into out_dir.  Spec keys:
// datasets [{kind, m, n, r, seed, path, name}], algorithms [names], inits_per_dataset,
// max_iterations, max_seconds (null = none), base_seed, threads, wall_timing.
int ref_suite_emit(const char* spec_json, const char* out_dir) {
  return guard([&] {
    const nlohmann::json j = nlohmann::json::parse(spec_json);
    enmf::SuiteSpec spec;
    for (const auto& d : j.at("datasets")) {
      enmf::DatasetSpec ds;
      const std::string kind = d.at("kind");
      ds.kind = kind == "lowrank" ? enmf::DatasetKind::lowrank
                : kind == "fullrank" ? enmf::DatasetKind::fullrank : enmf::DatasetKind::file;
      ds.m = d.value("m", 0);
      ds.n = d.value("n", 0);
      ds.r = d.value("r", 0);
      ds.seed = d.value("seed", 0);
      ds.path = d.value("path", std::string());
      ds.name = d.value("name", std::string());
      spec.datasets.push_back(ds);
    }
    for (const auto& a : j.at("algorithms")) spec.algorithms.push_back(enmf::make_algorithm(a.get<std::string>()));
    spec.inits_per_dataset = j.value("inits_per_dataset", 10);
    spec.budget.max_iterations = j.value("max_iterations", 100);
    if (j.contains("max_seconds") && !j.at("max_seconds").is_null()) spec.budget.max_seconds = j.at("max_seconds");
    spec.base_seed = j.value("base_seed", 1);
    spec.threads = j.value("threads", 1);
    spec.wall_timing = j.value("wall_timing", false);
    enmf::emit(enmf::run_suite(spec), out_dir);
  });
}

}  // extern "C"

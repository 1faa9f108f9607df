// io.cpp — host side of the data boundary: the reference's file formats and synthetic
// generators (enmf/data.hpp, enmf/rng.hpp), native and multi-threaded, behind the C-ABI.
//
//   Matrix Market coordinate real|integer general     data.hpp:159-240  (read), 242-257 (write)
//   headerless dense CSV                              data.hpp:262-309
//   per-run trace CSV                                 data.hpp:316-326
//   shortest round-trip number format                 data.hpp:101-105
//   lowrank_factors / gen_lowrank / gen_fullrank /
//   random_init / uniform_matrix / mix_seed           data.hpp:58-97, rng.hpp:30-57
//
// The readers parse the entry lines in parallel (one slice of the file per host thread,
// std::from_chars — the same correctly-rounded conversion the reference uses) and build the
// CSR arrays with a counting pass over rows.  Any slice that meets something other than a
// clean entry sends the whole file through the sequential reader, which reproduces the
// reference's first error, its message and its line number exactly (the error path is rare
// and never performance-relevant).  Writers format slices in parallel and write them in order.
// Compiled with -ffp-contract=off: gen_lowrank's product must round like the reference's
// (linalg.hpp:174-189, one multiply and one add per term, row-major accumulation order).
#include <algorithm>
#include <atomic>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <string_view>
#include <system_error>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/enmf_gpu.h"

namespace enmf_host {
void set_last_error(const std::string& msg);  // engine.cu: the thread-local message of enmf_gpu_last_error()
}

struct enmf_io_matrix {
  size_t rows = 0, cols = 0;
  bool sparse = false;
  std::vector<uint64_t> offsets, col_idx;
  std::vector<double> values;
};

namespace {

thread_local size_t g_err_line = 0;

struct IoFail {
  int code;
  std::string msg;
  size_t line;
};

[[noreturn]] void parse_fail(const std::string& what, size_t line) {
  // enmf::ParseError (data.hpp:34-43): the line is appended to the message when > 0
  throw IoFail{ENMF_PARSE_ERROR, line > 0 ? what + " (line " + std::to_string(line) + ")" : what, line};
}

template <class F>
int io_guard(F&& f) {
  try {
    g_err_line = 0;
    f();
    return ENMF_OK;
  } catch (const IoFail& e) {
    g_err_line = e.line;
    enmf_host::set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    enmf_host::set_last_error("out of host memory");
    return ENMF_IO_ERROR;
  } catch (const std::exception& e) {
    enmf_host::set_last_error(e.what());
    return ENMF_INVALID_ARGUMENT;
  }
}

unsigned host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return std::max(1u, std::min(h == 0 ? 1u : h, 64u));
}

template <class F>
void parallel_for(size_t parts, F&& f) {
  if (parts <= 1) {
    if (parts == 1) f(0);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(parts - 1);
  for (size_t p = 1; p < parts; ++p) pool.emplace_back([&, p] { f(p); });
  f(0);
  for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------- text helpers
// isspace in the "C" locale, as the reference's trim/next_token use it (data.hpp:109-127)
inline bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

std::string_view trim(std::string_view s) {
  while (!s.empty() && is_space(s.front())) s.remove_prefix(1);
  while (!s.empty() && is_space(s.back())) s.remove_suffix(1);
  return s;
}

bool next_token(std::string_view& s, std::string_view& tok) {
  size_t i = 0;
  while (i < s.size() && is_space(s[i])) ++i;
  if (i == s.size()) return false;
  size_t j = i;
  while (j < s.size() && !is_space(s[j])) ++j;
  tok = s.substr(i, j - i);
  s.remove_prefix(j);
  return true;
}

// non-throwing forms for the parallel path
inline bool to_double(std::string_view t, double& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}
inline bool to_index(std::string_view t, size_t& v) {
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  return r.ec == std::errc() && r.ptr == t.data() + t.size();
}
double parse_double(std::string_view t, size_t line) {
  double v = 0.0;
  if (!to_double(t, v)) parse_fail("malformed number '" + std::string(t) + "'", line);
  return v;
}
size_t parse_index(std::string_view t, size_t line) {
  size_t v = 0;
  if (!to_index(t, v)) parse_fail("malformed integer '" + std::string(t) + "'", line);
  return v;
}
std::string lower(std::string_view s) {
  std::string o(s);
  for (char& c : o) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return o;
}

// Lines exactly as std::getline splits them: on '\n', the last line may lack one, and a
// final '\n' does not start another line.
struct Lines {
  const char* p;
  const char* end;
  bool next(std::string_view& line) {
    if (p >= end) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
    const char* e = nl ? nl : end;
    line = std::string_view(p, (size_t)(e - p));
    p = nl ? nl + 1 : end;
    return true;
  }
};

std::string read_file(const char* path) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) throw IoFail{ENMF_IO_ERROR, std::string("cannot open '") + path + "' for reading", 0};
  std::string buf;
  char tmp[1 << 16];
  size_t got;
  if (std::fseek(f, 0, SEEK_END) == 0) {
    const long sz = std::ftell(f);
    if (sz > 0) buf.reserve((size_t)sz);
    std::fseek(f, 0, SEEK_SET);
  }
  while ((got = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.append(tmp, got);
  std::fclose(f);
  return buf;
}

// Slice [b, e) into about `parts` pieces that start at line beginnings.
std::vector<const char*> line_slices(const char* b, const char* e, size_t parts) {
  std::vector<const char*> cut{b};
  const size_t len = (size_t)(e - b);
  for (size_t k = 1; k < parts; ++k) {
    const char* c = b + len * k / parts;
    if (c <= cut.back()) continue;
    const char* nl = static_cast<const char*>(std::memchr(c - 1, '\n', (size_t)(e - (c - 1))));
    if (!nl || nl + 1 >= e) break;
    if (nl + 1 > cut.back()) cut.push_back(nl + 1);
  }
  cut.push_back(e);
  return cut;
}

constexpr size_t kParallelBytes = 1 << 20;  // below this a file is parsed on one thread

// ---------------------------------------------------------------- Matrix Market
struct Entry {
  size_t row, col;
  double value;
};

// Sequential reader of the entry lines (data.hpp:205-229): the exact error path.
void mm_entries_sequential(Lines ln, size_t lineno, size_t rows, size_t cols, size_t nnz,
                           std::vector<Entry>& entries) {
  entries.clear();
  entries.reserve(std::min<size_t>(nnz, 1 << 24));
  std::string_view line;
  while (entries.size() < nnz) {
    if (!ln.next(line))
      parse_fail("expected " + std::to_string(nnz) + " entries, found " + std::to_string(entries.size()), lineno);
    ++lineno;
    if (trim(line).empty()) continue;
    std::string_view rest = line, tok;
    next_token(rest, tok);
    const size_t i = parse_index(tok, lineno);
    if (!next_token(rest, tok)) parse_fail("entry missing column index", lineno);
    const size_t j = parse_index(tok, lineno);
    if (!next_token(rest, tok)) parse_fail("entry missing value", lineno);
    const double v = parse_double(tok, lineno);
    if (next_token(rest, tok)) parse_fail("trailing tokens on entry line", lineno);
    if (i < 1 || i > rows || j < 1 || j > cols)
      parse_fail("entry index (" + std::to_string(i) + ", " + std::to_string(j) + ") out of bounds", lineno);
    entries.push_back({i - 1, j - 1, v});
  }
  while (ln.next(line)) {
    ++lineno;
    if (!trim(line).empty()) parse_fail("unexpected content after last entry", lineno);
  }
}

// One slice of entry lines, no error reporting: false on anything but clean entries.
bool mm_entries_slice(const char* b, const char* e, size_t rows, size_t cols, std::vector<Entry>& out) {
  Lines ln{b, e};
  std::string_view line;
  while (ln.next(line)) {
    std::string_view rest = line, tok;
    if (!next_token(rest, tok)) continue;  // blank line
    size_t i, j;
    double v;
    if (!to_index(tok, i) || !next_token(rest, tok) || !to_index(tok, j) || !next_token(rest, tok) ||
        !to_double(tok, v) || next_token(rest, tok))
      return false;
    if (i < 1 || i > rows || j < 1 || j > cols) return false;
    out.push_back({i - 1, j - 1, v});
  }
  return true;
}

// SparseMatrix::from_triplets + validate (matrix.hpp:168-195, 226-250); their
// std::invalid_argument becomes a ParseError without a line (data.hpp:234-238).
void build_csr(size_t rows, size_t cols, const std::vector<Entry>& entries, enmf_io_matrix& m) {
  const size_t nnz = entries.size();
  m.rows = rows;
  m.cols = cols;
  m.sparse = true;
  m.offsets.assign(rows + 1, 0);
  for (const Entry& en : entries) ++m.offsets[en.row + 1];
  for (size_t i = 0; i < rows; ++i) m.offsets[i + 1] += m.offsets[i];
  std::vector<uint64_t> fill(m.offsets.begin(), m.offsets.end() - 1);
  std::vector<std::pair<uint64_t, double>> cv(nnz);
  for (const Entry& en : entries) cv[fill[en.row]++] = {en.col, en.value};
  // within-row order by column; then the first duplicate in (row, col) order, as the
  // reference's sort + adjacent scan finds it
  const size_t T = nnz >= (1u << 18) ? host_threads() : 1;
  std::vector<size_t> dup_row(T, SIZE_MAX), dup_col(T, 0);
  parallel_for(T, [&](size_t t) {
    const size_t r0 = rows * t / T, r1 = rows * (t + 1) / T;
    for (size_t i = r0; i < r1; ++i) {
      auto b = cv.begin() + (long)m.offsets[i], e = cv.begin() + (long)m.offsets[i + 1];
      std::sort(b, e, [](const auto& x, const auto& y) { return x.first < y.first; });
      for (auto p = b + (b != e ? 1 : 0); p < e; ++p)
        if (p->first == (p - 1)->first) {
          dup_row[t] = i;
          dup_col[t] = p->first;
          return;
        }
    }
  });
  for (size_t t = 0; t < T; ++t)
    if (dup_row[t] != SIZE_MAX)
      parse_fail("SparseMatrix: duplicate entry at (" + std::to_string(dup_row[t]) + ", " +
                     std::to_string(dup_col[t]) + ")",
                 0);
  m.col_idx.resize(nnz);
  m.values.resize(nnz);
  for (size_t p = 0; p < nnz; ++p) {
    m.col_idx[p] = cv[p].first;
    m.values[p] = cv[p].second;
    if (!std::isfinite(cv[p].second)) parse_fail("SparseMatrix: values must be finite", 0);
  }
}

void read_matrix_market(const char* path, enmf_io_matrix& out) {
  const std::string text = read_file(path);
  Lines ln{text.data(), text.data() + text.size()};
  std::string_view line;
  size_t lineno = 0;
  if (!ln.next(line)) parse_fail("empty file", 0);
  ++lineno;
  {
    std::string_view rest = line, banner, object, format, field, symmetry;
    if (!next_token(rest, banner) || lower(banner) != "%%matrixmarket")
      parse_fail("missing %%MatrixMarket banner", lineno);
    if (!next_token(rest, object) || !next_token(rest, format) || !next_token(rest, field) ||
        !next_token(rest, symmetry))
      parse_fail("banner needs object, format, field and symmetry", lineno);
    const std::string obj = lower(object), fmt = lower(format), fld = lower(field), sym = lower(symmetry);
    if (obj != "matrix") throw IoFail{ENMF_UNSUPPORTED_FORMAT, "unsupported object '" + obj + "'", 0};
    if (fmt != "coordinate") throw IoFail{ENMF_UNSUPPORTED_FORMAT, "unsupported format '" + fmt + "'", 0};
    if (fld != "real" && fld != "integer")
      throw IoFail{ENMF_UNSUPPORTED_FORMAT, "unsupported field '" + fld + "'", 0};
    if (sym != "general") throw IoFail{ENMF_UNSUPPORTED_FORMAT, "unsupported symmetry '" + sym + "'", 0};
  }
  size_t rows = 0, cols = 0, nnz = 0;
  for (;;) {  // size line: the first non-comment, non-blank line after the banner
    if (!ln.next(line)) parse_fail("missing size line", lineno);
    ++lineno;
    const std::string_view t = trim(line);
    if (t.empty() || t.front() == '%') continue;
    std::string_view rest = line, tok;
    if (!next_token(rest, tok)) parse_fail("missing row count", lineno);
    rows = parse_index(tok, lineno);
    if (!next_token(rest, tok)) parse_fail("missing column count", lineno);
    cols = parse_index(tok, lineno);
    if (!next_token(rest, tok)) parse_fail("missing entry count", lineno);
    nnz = parse_index(tok, lineno);
    if (next_token(rest, tok)) parse_fail("trailing tokens on size line", lineno);
    break;
  }
  if (rows == 0 || cols == 0) parse_fail("matrix dimensions must be positive", lineno);

  std::vector<Entry> entries;
  const char* body = ln.p;
  const char* end = ln.end;
  bool clean = false;
  if ((size_t)(end - body) >= kParallelBytes) {
    const auto cut = line_slices(body, end, host_threads());
    const size_t S = cut.size() - 1;
    std::vector<std::vector<Entry>> part(S);
    std::vector<char> ok(S, 0);
    parallel_for(S, [&](size_t s) { ok[s] = mm_entries_slice(cut[s], cut[s + 1], rows, cols, part[s]) ? 1 : 0; });
    size_t total = 0;
    clean = true;
    for (size_t s = 0; s < S; ++s) {
      clean = clean && ok[s];
      total += part[s].size();
    }
    if (clean && total == nnz) {
      entries.reserve(total);
      for (auto& p : part) entries.insert(entries.end(), p.begin(), p.end());
    } else {
      clean = false;
    }
  }
  if (!clean) mm_entries_sequential(ln, lineno, rows, cols, nnz, entries);
  build_csr(rows, cols, entries, out);
}

// ---------------------------------------------------------------- dense CSV
// One line of a dense CSV (data.hpp:268-290).  Throws the reference's errors when `line` > 0;
// with line == 0 returns false instead.
bool csv_line(std::string_view sv, size_t lineno, std::vector<double>& values, size_t& count) {
  if (!sv.empty() && sv.back() == '\r') sv.remove_suffix(1);
  count = 0;
  size_t start = 0;
  for (;;) {
    const size_t comma = sv.find(',', start);
    const std::string_view cell =
        trim(sv.substr(start, comma == std::string_view::npos ? comma : comma - start));
    if (cell.empty()) {
      if (lineno) parse_fail("empty cell", lineno);
      return false;
    }
    double v;
    if (!to_double(cell, v)) {
      if (lineno) parse_fail("malformed number '" + std::string(cell) + "'", lineno);
      return false;
    }
    values.push_back(v);
    ++count;
    if (comma == std::string_view::npos) break;
    start = comma + 1;
  }
  return true;
}

void csv_sequential(const std::string& text, enmf_io_matrix& out) {
  Lines ln{text.data(), text.data() + text.size()};
  std::string_view line;
  size_t rows = 0, cols = 0, lineno = 0, count = 0;
  out.values.clear();
  while (ln.next(line)) {
    ++lineno;
    csv_line(line, lineno, out.values, count);
    if (rows == 0) {
      cols = count;
    } else if (count != cols) {
      parse_fail("row has " + std::to_string(count) + " values, expected " + std::to_string(cols), lineno);
    }
    ++rows;
  }
  if (rows == 0) parse_fail("empty file", 0);
  out.rows = rows;
  out.cols = cols;
}

void read_dense_csv(const char* path, enmf_io_matrix& out) {
  const std::string text = read_file(path);
  out.sparse = false;
  bool clean = false;
  if (text.size() >= kParallelBytes) {
    const char* b = text.data();
    const char* e = b + text.size();
    const auto cut = line_slices(b, e, host_threads());
    const size_t S = cut.size() - 1;
    std::vector<std::vector<double>> part(S);
    std::vector<size_t> nrows(S, 0), width(S, 0);
    std::vector<char> ok(S, 1);
    parallel_for(S, [&](size_t s) {
      Lines ln{cut[s], cut[s + 1]};
      std::string_view line;
      size_t count = 0;
      while (ln.next(line)) {
        if (!csv_line(line, 0, part[s], count) || (nrows[s] > 0 && count != width[s])) {
          ok[s] = 0;
          return;
        }
        width[s] = count;
        ++nrows[s];
      }
    });
    clean = true;
    size_t rows = 0;
    for (size_t s = 0; s < S; ++s) {
      clean = clean && ok[s] && (nrows[s] == 0 || width[s] == width[0]);
      rows += nrows[s];
    }
    if (clean && rows > 0) {
      out.rows = rows;
      out.cols = width[0];
      out.values.clear();
      out.values.reserve(rows * out.cols);
      for (auto& p : part) out.values.insert(out.values.end(), p.begin(), p.end());
    } else {
      clean = false;
    }
  }
  if (!clean) csv_sequential(text, out);
  // DenseMatrix(rows, cols, values) (matrix.hpp:42-51): std::invalid_argument, not a ParseError
  for (double v : out.values)
    if (!std::isfinite(v)) throw IoFail{ENMF_INVALID_ARGUMENT, "DenseMatrix: values must be finite", 0};
}

// ---------------------------------------------------------------- writers
inline void put_double(std::string& s, double v) {
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);  // shortest round trip (data.hpp:101-105)
  s.append(buf, r.ptr);
}
inline void put_index(std::string& s, uint64_t v) {
  char buf[24];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  s.append(buf, r.ptr);
}

struct OutFile {
  std::FILE* f;
  std::string path;
  explicit OutFile(const char* p) : f(std::fopen(p, "wb")), path(p) {
    if (!f) throw IoFail{ENMF_IO_ERROR, "cannot open '" + path + "' for writing", 0};
  }
  void write(const std::string& s) {
    if (!s.empty() && std::fwrite(s.data(), 1, s.size(), f) != s.size())
      throw IoFail{ENMF_IO_ERROR, "write to '" + path + "' failed", 0};
  }
  void close() {
    const int rc = std::fclose(f);
    f = nullptr;
    if (rc != 0) throw IoFail{ENMF_IO_ERROR, "write to '" + path + "' failed", 0};
  }
  ~OutFile() {
    if (f) std::fclose(f);
  }
};

// Rows [0, rows) formatted by `fmt(row, string&)` on all host threads, written in order.
template <class F>
void write_rows(OutFile& out, size_t rows, size_t bytes_hint, F&& fmt) {
  const size_t T = bytes_hint >= kParallelBytes ? std::min<size_t>(host_threads(), std::max<size_t>(rows, 1)) : 1;
  const size_t block = std::max<size_t>(1, (rows + 4 * T - 1) / (4 * T));
  for (size_t base = 0; base < rows; base += block * T) {
    std::vector<std::string> part(T);
    parallel_for(T, [&](size_t t) {
      const size_t r0 = base + t * block, r1 = std::min(rows, r0 + block);
      for (size_t i = r0; i < r1; ++i) fmt(i, part[t]);
    });
    for (auto& p : part) out.write(p);
  }
}

void check_csr(const uint64_t* off, const uint64_t* cidx, const double* vals, size_t rows, size_t cols) {
  // SparseMatrix::validate (matrix.hpp:226-250)
  auto bad = [](const char* m) { throw IoFail{ENMF_INVALID_ARGUMENT, m, 0}; };
  if (rows == 0 || cols == 0) bad("SparseMatrix: rows and cols must be >= 1");
  if (!off || off[0] != 0) bad("SparseMatrix: inconsistent compressed storage");
  for (size_t i = 0; i < rows; ++i) {
    if (off[i] > off[i + 1]) bad("SparseMatrix: offsets must be non-decreasing");
    for (uint64_t p = off[i]; p < off[i + 1]; ++p) {
      if (cidx[p] >= cols) bad("SparseMatrix: column index out of range");
      if (p > off[i] && cidx[p] <= cidx[p - 1]) bad("SparseMatrix: column indices must be strictly increasing within a row");
      if (!std::isfinite(vals[p])) bad("SparseMatrix: values must be finite");
    }
  }
}

// ---------------------------------------------------------------- generators
void fill_uniform(std::mt19937_64& g, double* p, size_t n) {
  for (size_t i = 0; i < n; ++i) p[i] = static_cast<double>(g() >> 11) * 0x1.0p-53;  // rng.hpp:47-49
}
size_t checked_size(size_t rows, size_t cols) {
  if (rows == 0 || cols == 0) throw IoFail{ENMF_INVALID_ARGUMENT, "DenseMatrix: rows and cols must be >= 1", 0};
  if (cols > SIZE_MAX / rows) throw IoFail{ENMF_INVALID_ARGUMENT, "DenseMatrix: shape overflows size_t", 0};
  return rows * cols;
}

}  // namespace

extern "C" {

size_t enmf_gpu_last_error_line(void) { return g_err_line; }

int enmf_io_read_matrix_market(const char* path, enmf_io_matrix** out) {
  return io_guard([&] {
    if (!path || !out) throw IoFail{ENMF_INVALID_ARGUMENT, "null argument", 0};
    auto m = std::make_unique<enmf_io_matrix>();
    read_matrix_market(path, *m);
    *out = m.release();
  });
}

int enmf_io_read_dense_csv(const char* path, enmf_io_matrix** out) {
  return io_guard([&] {
    if (!path || !out) throw IoFail{ENMF_INVALID_ARGUMENT, "null argument", 0};
    auto m = std::make_unique<enmf_io_matrix>();
    read_dense_csv(path, *m);
    *out = m.release();
  });
}

void enmf_io_matrix_shape(const enmf_io_matrix* a, size_t* rows, size_t* cols, size_t* nnz, int* is_sparse) {
  if (!a) return;
  if (rows) *rows = a->rows;
  if (cols) *cols = a->cols;
  if (nnz) *nnz = a->values.size();
  if (is_sparse) *is_sparse = a->sparse ? 1 : 0;
}
const uint64_t* enmf_io_matrix_offsets(const enmf_io_matrix* a) { return a && a->sparse ? a->offsets.data() : nullptr; }
const uint64_t* enmf_io_matrix_col_indices(const enmf_io_matrix* a) {
  return a && a->sparse ? a->col_idx.data() : nullptr;
}
const double* enmf_io_matrix_values(const enmf_io_matrix* a) { return a ? a->values.data() : nullptr; }
void enmf_io_matrix_free(enmf_io_matrix* a) { delete a; }

int enmf_io_write_matrix_market(const char* path, const uint64_t* offsets, const uint64_t* col_idx,
                                const double* vals, size_t rows, size_t cols) {
  return io_guard([&] {
    if (!path) throw IoFail{ENMF_INVALID_ARGUMENT, "null argument", 0};
    check_csr(offsets, col_idx, vals, rows, cols);
    const size_t nnz = offsets[rows];
    OutFile out(path);
    std::string head = "%%MatrixMarket matrix coordinate real general\n";
    put_index(head, rows);
    head += ' ';
    put_index(head, cols);
    head += ' ';
    put_index(head, nnz);
    head += '\n';
    out.write(head);
    write_rows(out, rows, nnz * 24, [&](size_t i, std::string& s) {
      for (uint64_t p = offsets[i]; p < offsets[i + 1]; ++p) {
        put_index(s, i + 1);
        s += ' ';
        put_index(s, col_idx[p] + 1);
        s += ' ';
        put_double(s, vals[p]);
        s += '\n';
      }
    });
    out.close();
  });
}

int enmf_io_write_dense_csv(const char* path, const double* x, size_t rows, size_t cols) {
  return io_guard([&] {
    if (!path || !x) throw IoFail{ENMF_INVALID_ARGUMENT, "null argument", 0};
    checked_size(rows, cols);
    OutFile out(path);
    write_rows(out, rows, rows * cols * 20, [&](size_t i, std::string& s) {
      const double* row = x + i * cols;
      for (size_t j = 0; j < cols; ++j) {
        if (j > 0) s += ',';
        put_double(s, row[j]);
      }
      s += '\n';
    });
    out.close();
  });
}

int enmf_io_write_run_csv(const char* path, const enmf_gpu_iter* iters, size_t n, double e_min) {
  return io_guard([&] {
    if (!path || (!iters && n)) throw IoFail{ENMF_INVALID_ARGUMENT, "null argument", 0};
    OutFile out(path);
    std::string s = "iter,elapsed_s,rel_err,E,beta,restarted\n";
    for (size_t k = 0; k < n; ++k) {
      const enmf_gpu_iter& it = iters[k];
      put_index(s, it.iteration);
      s += ',';
      put_double(s, it.elapsed_seconds);
      s += ',';
      put_double(s, it.relative_error);
      s += ',';
      put_double(s, it.relative_error - e_min);
      s += ',';
      put_double(s, it.beta);
      s += ',';
      s += it.restarted ? '1' : '0';
      s += '\n';
    }
    out.write(s);
    out.close();
  });
}

size_t enmf_io_format_double(double v, char* buf, size_t cap) {
  char tmp[32];
  const auto r = std::to_chars(tmp, tmp + sizeof tmp, v);
  const size_t len = (size_t)(r.ptr - tmp);
  if (buf && cap > 0) {
    const size_t k = std::min(len, cap - 1);
    std::memcpy(buf, tmp, k);
    buf[k] = '\0';
  }
  return len;
}

uint64_t enmf_mix_seed(uint64_t base, uint64_t a, uint64_t b) {
  auto mix64 = [](uint64_t z) {  // rng.hpp:30-34
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  const uint64_t g = 0x9E3779B97F4A7C15ull;  // rng.hpp:36-42
  uint64_t h = mix64(base + g);
  h = mix64(h ^ (a + g));
  return mix64(h ^ (b + g));
}

int enmf_uniform_matrix(size_t rows, size_t cols, uint64_t seed, double* out) {
  return io_guard([&] {
    const size_t n = checked_size(rows, cols);
    if (!out) throw IoFail{ENMF_INVALID_ARGUMENT, "null argument", 0};
    std::mt19937_64 g(seed);
    fill_uniform(g, out, n);
  });
}

int enmf_random_init(size_t m, size_t n, size_t r, uint64_t seed, double* w, double* h) {
  return io_guard([&] {
    const size_t ws = checked_size(m, r), hs = checked_size(r, n);
    if (!w || !h) throw IoFail{ENMF_INVALID_ARGUMENT, "null argument", 0};
    std::mt19937_64 g(seed);  // data.hpp:90-97: W then H from one stream
    fill_uniform(g, w, ws);
    fill_uniform(g, h, hs);
  });
}

int enmf_lowrank_factors(size_t m, size_t n, size_t r, uint64_t seed, double* w, double* h) {
  if (r == 0 || r > std::min(m, n)) {  // data.hpp:61-65
    enmf_host::set_last_error("lowrank_factors: need 1 <= r <= min(m, n)");
    return ENMF_INVALID_ARGUMENT;
  }
  return enmf_random_init(m, n, r, seed, w, h);
}

int enmf_gen_lowrank(size_t m, size_t n, size_t r, uint64_t seed, double* x) {
  if (!x) {
    enmf_host::set_last_error("null argument");
    return ENMF_INVALID_ARGUMENT;
  }
  if (r == 0 || r > std::min(m, n)) {
    enmf_host::set_last_error("lowrank_factors: need 1 <= r <= min(m, n)");
    return ENMF_INVALID_ARGUMENT;
  }
  return io_guard([&] {
    std::vector<double> w(checked_size(m, r)), h(checked_size(r, n));
    checked_size(m, n);
    std::mt19937_64 g(seed);
    fill_uniform(g, w.data(), w.size());
    fill_uniform(g, h.data(), h.size());
    // multiply (linalg.hpp:174-189): out(i,:) += w(i,p)·h(p,:) for p ascending; rows in parallel
    const size_t T = m * n * r >= (1u << 22) ? std::min<size_t>(host_threads(), m) : 1;
    parallel_for(T, [&](size_t t) {
      for (size_t i = m * t / T; i < m * (t + 1) / T; ++i) {
        double* oi = x + i * n;
        std::fill(oi, oi + n, 0.0);
        for (size_t p = 0; p < r; ++p) {
          const double a = w[i * r + p];
          const double* bp = h.data() + p * n;
          for (size_t j = 0; j < n; ++j) oi[j] += a * bp[j];
        }
      }
    });
  });
}

int enmf_gen_fullrank(size_t m, size_t n, uint64_t seed, double* x) { return enmf_uniform_matrix(m, n, seed, x); }

// BASELINE configs[4] (C5) data, X = W0·H0 + 0.01·|N(0,1)| on T×T tiles with per-tile streams, so
// any rank can build any block of the same matrix and the result is identical for any thread
// count (the stream layout of oracle/replica.c orc_gen_tiled, which the tests pin bitwise):
//   W0 row block bi: uniform, row-major, mt19937_64(mix_seed(seed, 1, bi));
//   H0 column block bj: uniform, for k: for j in the block, mt19937_64(mix_seed(seed, 2, bj));
//   X tile (bi, bj): Σ_k W0(i,k)·H0(k,j) (k ascending from 0.0) + 0.01·|Box–Muller normal|, one
//   normal per entry row-major in the tile, mt19937_64(mix_seed(seed, 3, bi·nbj + bj)).
// Writes the block rows [row0, row0+rows) × columns [col0, col0+cols) into x (row stride cols).
int enmf_gen_tiled(size_t m, size_t n, size_t r, uint64_t seed, size_t T, size_t row0, size_t rows, size_t col0,
                   size_t cols, double* x) {
  return io_guard([&] {
    if (!x) throw IoFail{ENMF_INVALID_ARGUMENT, "null argument", 0};
    if (T == 0) T = 4096;
    if (row0 + rows > m || col0 + cols > n || rows == 0 || cols == 0 || r == 0)
      throw IoFail{ENMF_INVALID_ARGUMENT, "gen_tiled: block outside the matrix", 0};
    const size_t nbj = (n + T - 1) / T;
    const size_t bi0 = row0 / T, bi1 = (row0 + rows - 1) / T, bj0 = col0 / T, bj1 = (col0 + cols - 1) / T;
    const size_t ni = bi1 - bi0 + 1, nj = bj1 - bj0 + 1;
    std::vector<double> w(ni * T * r), h(r * nj * T);   // the W0 row blocks / H0 column blocks touched
    parallel_for(std::min<size_t>(host_threads(), ni + nj), [&](size_t t) {
      const size_t P = std::min<size_t>(host_threads(), ni + nj);
      for (size_t q = t; q < ni + nj; q += P) {
        if (q < ni) {
          const size_t bi = bi0 + q, i1 = std::min(m, (bi + 1) * T);
          std::mt19937_64 g(enmf_mix_seed(seed, 1, bi));
          for (size_t i = bi * T; i < i1; ++i)
            for (size_t k = 0; k < r; ++k) w[((i - bi0 * T)) * r + k] = static_cast<double>(g() >> 11) * 0x1.0p-53;
        } else {
          const size_t bj = bj0 + (q - ni), j1 = std::min(n, (bj + 1) * T);
          std::mt19937_64 g(enmf_mix_seed(seed, 2, bj));
          for (size_t k = 0; k < r; ++k)
            for (size_t j = bj * T; j < j1; ++j) h[k * (nj * T) + (j - bj0 * T)] = static_cast<double>(g() >> 11) * 0x1.0p-53;
        }
      }
    });
    const size_t tiles = ni * nj, P = std::min<size_t>(host_threads(), tiles);
    parallel_for(P, [&](size_t t) {
      std::vector<double> rowbuf(T);
      for (size_t q = t; q < tiles; q += P) {
        const size_t bi = bi0 + q / nj, bj = bj0 + q % nj;
        const size_t ti0 = bi * T, ti1 = std::min(m, ti0 + T), tj0 = bj * T, tj1 = std::min(n, tj0 + T);
        std::mt19937_64 g(enmf_mix_seed(seed, 3, bi * nbj + bj));
        auto unif = [&g] { return static_cast<double>(g() >> 11) * 0x1.0p-53; };
        for (size_t i = ti0; i < ti1; ++i) {
          const bool keep_row = i >= row0 && i < row0 + rows;
          // the tile's normals are drawn row by row whether or not this block keeps the row
          for (size_t j = tj0; j < tj1; ++j) {
            const double u1 = unif(), u2 = unif();
            rowbuf[j - tj0] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
          }
          if (!keep_row) continue;
          const double* wi = w.data() + (i - bi0 * T) * r;
          const size_t c0 = std::max(tj0, col0), c1 = std::min(tj1, col0 + cols);
          double* xo = x + (i - row0) * cols - col0;
          for (size_t j = c0; j < c1; ++j) xo[j] = 0.0;
          for (size_t k = 0; k < r; ++k) {
            const double a = wi[k];
            const double* hk = h.data() + k * (nj * T) - bj0 * T;
            for (size_t j = c0; j < c1; ++j) xo[j] += a * hk[j];
          }
          for (size_t j = c0; j < c1; ++j) xo[j] += 0.01 * std::fabs(rowbuf[j - tj0]);
        }
      }
    });
  });
}

}  // extern "C"

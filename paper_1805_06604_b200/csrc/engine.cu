// engine.cu — host driver and C-ABI of the B200 enmf hot path.
//
// Replays enmf::run / enmf::step (engine.hpp:309-521) with every decision
// taken on the device (DevState), so one outer iteration is one CUDA graph:
//
//   iter_begin → gram(W_y)+reinit → W_yᵀX → [HALS sweeps: WHILE node | BPP]
//   → (hp≥2) H extrapolation → gram(T)+reinit → T·Xᵀ → [HALS | BPP]
//   → (literal hp1) fresh H_y products → gram(W_n), <W_n, X Tᵀ> → decide → finalize
//
// The host only launches the instantiated graph K times and reads the
// records back at the end (no per-iteration or per-sweep synchronisation).
// Device layouts: X row-major m×n as given; W kept
// transposed (Wᵀ, r×m) so the W update sweeps contiguous rows and the X·Tᵀ
// GEMM writes its result straight into the r×m layout the sweep consumes;
// H r×n as given.  W is transposed only at entry and exit.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "bpp.cuh"
#include "batch.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "hals.cuh"
#include "hals_tm.cuh"
#include "misc.cuh"
#include "sparse.cuh"
#include "ozaki.cuh"
#include "ozk.cuh"
#include "tf32k.cuh"
#include "sweep_tf32.cuh"
#include "hals_rl.cuh"

namespace {

thread_local std::string g_last_error;

struct Fail {
  int code;
  std::string msg;
};

#define CU(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      throw Fail{ENMF_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
    }                                                                                \
  } while (0)

#define CUK() CU(cudaGetLastError())

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t cnt) {
    if (cnt <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    CU(cudaMalloc(&p, std::max<size_t>(cnt, 1) * sizeof(T)));
    n = cnt;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

constexpr int kSMs = 148;  // B200; refreshed from the device at context creation

}  // namespace

struct enmf_gpu_ctx {
  int device = 0;
  int sms = kSMs;
  cudaStream_t stream = nullptr, body_stream = nullptr;
  unsigned long long launches = 0;
  // data matrix
  DBuf<double> x_own;
  const double* x = nullptr;
  size_t m = 0, n = 0;
  // host X in flight (x_upload_async .. x_join .. x_verdict): the copy runs on its own stream so
  // that begin()'s allocations and factor upload overlap it; 0 = none, 1 = copy enqueued, not yet
  // joined by the engine stream, 2 = joined, finite check enqueued, verdict not read
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t x_copied = nullptr, x_checked = nullptr;
  int* x_bad = nullptr;                    // pinned host flag
  int x_state = 0;
  // CSR data matrix (enmf_gpu_load_csr): CSR for X·Tᵀ, CSC copy for W_yᵀX
  bool sparse = false;
  size_t nnz = 0;
  DBuf<long long> csr_ptr, csc_ptr;
  // fixed-size chunks of the CSR rows / CSC columns for the FP64-mode gathers (sparse.cuh)
  struct Chunks {
    DBuf<int> line, slot, mline, mfirst, mcount;
    DBuf<long long> beg, end;
    int n = 0, nmulti = 0, nslots = 0;
  } ch_csr, ch_csc;
  DBuf<double> chunk_part;
  DBuf<int> csr_idx, csc_idx;
  DBuf<double> csr_val, csc_val, rowmaj;
  // FP64 cross products on INT8 tensor cores (ozaki.cuh): X digits (cut once per load)
  struct XDig {                            // digits of one X operand (full X, or a rank's block)
    DBuf<int8_t> d;
    DBuf<int> e;
    DBuf<int> sums;                        // digit sums along the contracted index, SMAX × N
    const double* src = nullptr;
    long rows = 0, cols = 0;
    bool ready = false, by_row = false;
    int levels = 6;                        // digit levels used (ozk's S)
    long N = 0, K = 0;                     // digit operand: N rows (output columns) × K contracted
  } xd_xt, xd_x, xd_cols, xd_rows;          // one GPU: X scaled per row (T·Xᵀ) / per column (W_yᵀX)
  DBuf<double> ozws;                       // ozk unit partials
  DBuf<int8_t> adig;
  DBuf<int> aexp, asum;
  DBuf<unsigned long long> amax;
  DBuf<double> opart;
  // TF32 variant: FP32 copy of X (once per load), FP32 factor / product staging
  bool xf_ready = false;
  DBuf<float> xf, af, cf;
  // factors and products
  DBuf<double> WT, WyT, WnT, H, Hy, Hn, CH, P, Plit, GH, GW, GWn, Glit, scratch, Gf;
  DBuf<double> partials, gain_part, terms, ddpart, dd;
  DBuf<int> part_nf, flags, kpart_nf;
  DBuf<unsigned> counters;
  DBuf<double> kpartials;                 // kernel-level API calls: own split-K scratch (never a session graph's)
  DBuf<unsigned> kcounters;
  bool kapi = false;
  DBuf<unsigned long long> bpp_exch;
  DBuf<int> bpp_rounds, bpp_nf;
  DBuf<double> cmax;
  DBuf<DevState> st;
  DBuf<enmf_gpu_iter> recs;
  // instrumentation of the last solve
  int static_kernels = 0, kernels_per_sweep = 0;
  // open run session (enmf_gpu_begin .. enmf_gpu_end)
  struct Session* sess = nullptr;
  // multi-GPU sharding (enmf_gpu_dist_*); null or !ready = single GPU
  struct DistHost* dist = nullptr;
  // standalone kernel API
  int kernel_precision = ENMF_PRECISION_FP64;
  DBuf<double> ka, kb, kc, kd, ke, kf;
  DBuf<double> ls_part, ls_val;   // optimal_beta_linesearch scratch (never captured in a graph)
  DBuf<HalsCtl> kctl;
};

// Sharded (multi-GPU) state of a context, SURVEY §8(e).  The IPC-shared block
// of every rank holds [flags | slots | W_yᵀ replica r×m | T replica r×n].
struct DistHost {
  int rank = 0, world = 1;
  size_t m = 0, n = 0, r = 0;
  size_t row0 = 0, mp = 0, col0 = 0, np = 0;
  size_t slot = 0;                       // doubles per mailbox slot
  char* shared = nullptr;                // own block (cudaMalloc, IPC-exported)
  size_t shared_bytes = 0;
  char* peer[dist::MAXP] = {};           // every rank's block (own included)
  dist::View* dview = nullptr;           // device copy of the view
  unsigned long long* epoch = nullptr;
  int* err = nullptr;
  double* scratch = nullptr;
  DBuf<double> xc_own, xr_own;
  const double* xc = nullptr;            // X[:, col0:col0+np]  (m × np)
  const double* xr = nullptr;            // X[row0:row0+mp, :]  (mp × n)
  bool ready = false;

  static size_t header_bytes() { return 256; }
  size_t slots_bytes() const { return 2 * dist::MAXP * slot * sizeof(double); }
  double* wfull(int q) const { return reinterpret_cast<double*>(peer[q] + header_bytes() + slots_bytes()); }
  double* tfull(int q) const { return wfull(q) + r * m; }
};

// Balanced contiguous blocks: the first (len % world) ranks get one more.
inline void shard_bounds(size_t len, int rank, int world, size_t* off, size_t* cnt) {
  const size_t base = len / world, extra = len % world;
  *cnt = base + ((size_t)rank < extra ? 1 : 0);
  *off = (size_t)rank * base + std::min<size_t>((size_t)rank, extra);
}

namespace {

void set_attrs_once() {
  static bool done = false;
  if (done) return;
  auto big = [](const void* f, int bytes) {
    CU(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  };
#define GEMM_ATTR(W)                                                               \
  big((const void*)gemm::gemm_f64_dmma<false, 2, false, W>, gemm::SMEM_BYTES);     \
  big((const void*)gemm::gemm_f64_dmma<false, 2, true, W>, gemm::SMEM_BYTES);      \
  big((const void*)gemm::gemm_f64_dmma<false, 1, false, W>, gemm::SMEM_BYTES);     \
  big((const void*)gemm::gemm_f64_dmma<false, 1, true, W>, gemm::SMEM_BYTES);      \
  big((const void*)gemm::gemm_f64_dmma<true, 2, false, W>, gemm::SMEM_BYTES);      \
  big((const void*)gemm::gemm_f64_dmma<true, 2, true, W>, gemm::SMEM_BYTES);       \
  big((const void*)gemm::gemm_f64_dmma<true, 1, false, W>, gemm::SMEM_BYTES);      \
  big((const void*)gemm::gemm_f64_dmma<true, 1, true, W>, gemm::SMEM_BYTES);
  GEMM_ATTR(2)
  GEMM_ATTR(4)
#undef GEMM_ATTR
  big((const void*)gemm::gemm_f64_dmma_s<false, 2, false>, gemm::st::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_s<false, 2, true>, gemm::st::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_s<false, 1, false>, gemm::st::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_s<false, 1, true>, gemm::st::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_s<true, 2, false>, gemm::st::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_s<true, 2, true>, gemm::st::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_s<true, 1, false>, gemm::st::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_s<true, 1, true>, gemm::st::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_t<false, false>, gemm::tm::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_t<false, true>, gemm::tm::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_t<true, false>, gemm::tm::SMEM_BYTES);
  big((const void*)gemm::gemm_f64_dmma_t<true, true>, gemm::tm::SMEM_BYTES);
  big((const void*)hals::sweep_ws<32>, hals::ws_smem_bytes<32>());
  big((const void*)hals::sweep_ws<64>, hals::ws_smem_bytes<64>());
  big((const void*)hals::sweep_ws<128>, hals::ws_smem_bytes<128>());
  big((const void*)hals::sweep_ws<32, true>, hals::ws_smem_bytes<32>());
  big((const void*)hals::sweep_ws<64, true>, hals::ws_smem_bytes<64>());
  big((const void*)hals::sweep_ws<128, true>, hals::ws_smem_bytes<128>());
  big((const void*)hals::sweep_tm<128>, hals::tm_smem_bytes<128>());
  big((const void*)batch::run<8>, batch::smem_bytes());
  big((const void*)batch::run<16>, batch::smem_bytes());
  big((const void*)batch::run<24>, batch::smem_bytes());
  big((const void*)batch::run<32>, batch::smem_bytes());
  big((const void*)hals::sweep_fast<16, 1>, hals::smem_bytes<16, 1>());
  big((const void*)hals::sweep_fast<32, 1>, hals::smem_bytes<32, 1>());
  big((const void*)hals::sweep_fast<32, 2>, hals::smem_bytes<32, 2>());
  big((const void*)hals::sweep_fast<32, 4>, hals::smem_bytes<32, 4>());
  big((const void*)bpp::solve<32, 8>, bpp::smem_bytes<32, 8>());
  big((const void*)bpp::solve_fast<8>, bpp::fast_smem_bytes<8>());
  big((const void*)bpp::solve<64, 4>, bpp::smem_bytes<64, 4>());
  big((const void*)bpp::solve<128, 1>, bpp::smem_bytes<128, 1>());
  done = true;
}

inline unsigned grid_for(long count, int nt = 256, int maxb = 148 * 8) {
  long b = (count + nt - 1) / nt;
  return (unsigned)std::max<long>(1, std::min<long>(b, maxb));
}

// ---- precision modes ---------------------------------------------------------
enum { PREC_FAST = ENMF_PRECISION_FP64, PREC_TF32 = ENMF_PRECISION_TF32, PREC_EXACT = 2 };

// ---- contractions --------------------------------------------------------------
// Split-K factor: the smallest S whose CTA count fills the SMs to >= 95%
// (1 CTA/SM: 216 KB of shared memory).  Multi-tile GEMMs are capped at S = 8
// (partials cost 2·S·M·N·8 bytes of extra traffic; the last CTA of a tile
// reduces them); a single-tile GEMM (the r×r Gram) splits up to one CTA per
// SM with a separate fixed-order reduction.
int choose_splits(int tiles, int kblocks, int sms) {
  if (tiles >= 8 * sms) return 1;
  const int smax = tiles > 8 ? std::max(1, std::min(kblocks / 4, 8))
                             : std::max(1, std::min(kblocks / 4, sms));
  int best = 1;
  double best_eff = -1.0;
  for (int s = 1; s <= smax; ++s) {
    const long ctas = (long)tiles * s;
    const long waves = (ctas + sms - 1) / sms;
    const double eff = (double)ctas / (double)(waves * sms);
    if (eff >= 0.95) return s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

// C[M×N] = A[M×K] · op(B);  bk: B is N×K (K contiguous) else K×N (N contiguous).
bool gemm_big_tile() {  // ENMF_GEMM_TILE=128: the 128×128 single-CTA-per-SM kernel
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("ENMF_GEMM_TILE");
    v = (e && std::string(e) == "128") ? 1 : 0;
  }
  return v == 1;
}

// ---- TMA descriptors (cuTensorMapEncodeTiled through the runtime's driver entry point) ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      throw Fail{ENMF_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable"};
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// 2-D FP64 operand (outer rows of `inner` contiguous doubles, row stride ld) in boxes of
// box_inner × box_outer, SWIZZLE_128B (box_inner = 16 doubles = one 128-byte row), zeros past the edges
CUtensorMap f64_tmap(const double* base, long inner, long outer, long ld, int box_inner, int box_outer) {
  CUtensorMap m;
  const cuuint64_t dim[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t stride[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dim, stride, box,
                                    es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Fail{ENMF_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  return m;
}

// ENMF_GEMM_LOAD=cpasync: the FP64 DMMA GEMM loads its tiles with cp.async (gemm_f64_dmma_s)
// instead of TMA (gemm_f64_dmma_t) — A/B timing.
bool gemm_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("ENMF_GEMM_LOAD");
    v = (e && std::string(e) == "cpasync") ? 0 : 1;
  }
  return v == 1;
}

// Split-K scratch of one GEMM (the tile grid and split count gemm_launch_small / gemm_launch choose).
struct SplitNeed {
  int S, tiles;
  bool last;
};
SplitNeed split_need(const enmf_gpu_ctx* c, int M, int N, int K) {
  SplitNeed n{};
  if (!gemm_big_tile()) {
    n.tiles = ((N + gemm::st::BN - 1) / gemm::st::BN) * ((M + gemm::st::BM - 1) / gemm::st::BM);
    n.S = choose_splits(n.tiles, (K + gemm::st::BK - 1) / gemm::st::BK, 3 * c->sms);
  } else {
    n.tiles = ((N + gemm::BN - 1) / gemm::BN) * ((M + gemm::BM - 1) / gemm::BM);
    n.S = choose_splits(n.tiles, (K + gemm::BK - 1) / gemm::BK, c->sms);
  }
  n.last = n.S > 1 && n.S <= 8;
  return n;
}

// The split-K workspace for a launch: sized in begin() for every GEMM a session graph holds
// (presize_splits), so a captured launch never reallocates it — growing it while a stream is
// capturing would free memory an earlier node of the same graph still uses, hence an internal
// error.  Kernel-level API calls (c->kapi) use their own workspace, never a session graph's.
void split_ws(enmf_gpu_ctx* c, cudaStream_t s, const SplitNeed& n, int M, int N, double** part, unsigned** cnt) {
  DBuf<double>& P = c->kapi ? c->kpartials : c->partials;
  DBuf<unsigned>& Q = c->kapi ? c->kcounters : c->counters;
  if (n.S > 1) {
    const size_t need = (size_t)n.S * M * N;
    const bool grow = P.n < need || (n.last && Q.n < (size_t)n.tiles);
    if (grow) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      CU(cudaStreamIsCapturing(s, &cs));
      if (cs != cudaStreamCaptureStatusNone)
        throw Fail{ENMF_CUDA_ERROR, "internal: split-K workspace would grow during graph capture"};
    }
    P.ensure(need);
    if (n.last && Q.n < (size_t)n.tiles) {
      Q.ensure(n.tiles);
      CU(cudaMemsetAsync(Q.p, 0, sizeof(unsigned) * n.tiles, s));
    }
  }
  *part = n.S > 1 ? P.p : nullptr;
  *cnt = Q.p;
}

// Sizes the session workspace for the GEMMs of an m×n, rank-r problem held as ml rows / nl
// columns here (sharded: local extents): the two Grams (K = ml, nl) and both cross products on the
// DMMA GEMM (N = nl, K = m and N = ml, K = n; the INT8-digit / CSR / TF32 products use their own
// buffers).
void presize_splits(enmf_gpu_ctx* c, cudaStream_t s, size_t m, size_t n, size_t ml, size_t nl, size_t r) {
  size_t need = 0, tiles = 0;
  const int shapes[4][3] = {{(int)r, (int)r, (int)ml}, {(int)r, (int)r, (int)nl}, {(int)r, (int)nl, (int)m},
                            {(int)r, (int)ml, (int)n}};
  for (const auto& sh : shapes) {
    const SplitNeed k = split_need(c, sh[0], sh[1], sh[2]);
    if (k.S > 1) need = std::max(need, (size_t)k.S * sh[0] * sh[1]);
    if (k.last) tiles = std::max(tiles, (size_t)k.tiles);
  }
  if (need) c->partials.ensure(need);
  if (tiles && c->counters.n < tiles) {
    c->counters.ensure(tiles);
    CU(cudaMemsetAsync(c->counters.p, 0, sizeof(unsigned) * tiles, s));
  }
}

void gemm_launch_small(enmf_gpu_ctx* c, cudaStream_t s, bool bk, const double* A, long lda, const double* B, long ldb,
                       double* C, long ldc, int M, int N, int K, bool sym, const DevState* st) {
  using namespace gemm;
  const int tn = (N + st::BN - 1) / st::BN, tm = (M + st::BM - 1) / st::BM;
  const SplitNeed need = split_need(c, M, N, K);
  const int S = need.S;
  const bool last = need.last;
  double* part;
  unsigned* cnt;
  split_ws(c, s, need, M, N, &part, &cnt);
  const bool vec2 = (lda % 2 == 0) && (ldb % 2 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0);
  Params p{A, lda, B, ldb, C, ldc, M, N, K, S, part, cnt, sym ? 1 : 0, st};
  // M-tiles vary fastest (blockIdx.x): the r/64 CTAs sharing one X tile run
  // together, so X is fetched from HBM once and hit in L2 by the others.
  dim3 grid(tm, tn, S);
  if (vec2 && gemm_tma()) {   // TMA-fed (16-byte aligned bases and row strides)
    const CUtensorMap ta = f64_tmap(A, K, M, lda, 16, 64);
    const CUtensorMap tb = bk ? f64_tmap(B, K, N, ldb, 16, 64) : f64_tmap(B, N, K, ldb, 16, 16);
#define GEMM_GO_T(BKM, L) gemm_f64_dmma_t<BKM, L><<<grid, st::NTH, gemm::tm::SMEM_BYTES, s>>>(p, ta, tb)
    if (bk) { if (last) GEMM_GO_T(true, true); else GEMM_GO_T(true, false); }
    else { if (last) GEMM_GO_T(false, true); else GEMM_GO_T(false, false); }
#undef GEMM_GO_T
    CUK();
    c->launches++;
    if (S > 1 && !last) {
      reduce_splits<<<grid_for((long)M * N), 256, 0, s>>>(part, S, M, N, C, ldc, sym ? 1 : 0, st);
      CUK();
      c->launches++;
    }
    return;
  }
#define GEMM_GO(BKM, V, L) gemm_f64_dmma_s<BKM, V, L><<<grid, st::NTH, st::SMEM_BYTES, s>>>(p)
  if (bk) {
    if (vec2) { if (last) GEMM_GO(true, 2, true); else GEMM_GO(true, 2, false); }
    else { if (last) GEMM_GO(true, 1, true); else GEMM_GO(true, 1, false); }
  } else {
    if (vec2) { if (last) GEMM_GO(false, 2, true); else GEMM_GO(false, 2, false); }
    else { if (last) GEMM_GO(false, 1, true); else GEMM_GO(false, 1, false); }
  }
#undef GEMM_GO
  CUK();
  c->launches++;
  if (S > 1 && !last) {
    reduce_splits<<<grid_for((long)M * N), 256, 0, s>>>(part, S, M, N, C, ldc, sym ? 1 : 0, st);
    CUK();
    c->launches++;
  }
}

void gemm_launch(enmf_gpu_ctx* c, cudaStream_t s, bool bk, const double* A, long lda, const double* B, long ldb,
                 double* C, long ldc, int M, int N, int K, bool sym, const DevState* st) {
  using namespace gemm;
  if (!gemm_big_tile()) {
    gemm_launch_small(c, s, bk, A, lda, B, ldb, C, ldc, M, N, K, sym, st);
    return;
  }
  const int tn = (N + BN - 1) / BN, tm = (M + BM - 1) / BM;
  const SplitNeed need = split_need(c, M, N, K);
  const int S = need.S;
  const bool last = need.last;
  double* part;
  unsigned* cnt;
  split_ws(c, s, need, M, N, &part, &cnt);
  const bool vec2 = (lda % 2 == 0) && (ldb % 2 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0);
  Params p{A, lda, B, ldb, C, ldc, M, N, K, S, part, cnt, sym ? 1 : 0, st};
  dim3 grid(tn, tm, S);
  static int w16 = -1;  // ENMF_GEMM_WARPS=16: 16 warps of 32×32 instead of 8 of 64×32
  if (w16 < 0) {
    const char* e = std::getenv("ENMF_GEMM_WARPS");
    w16 = (e && std::string(e) == "16") ? 1 : 0;
  }
#define GEMM_GO(BKM, V, L)                                                                \
  do {                                                                                    \
    if (w16) gemm_f64_dmma<BKM, V, L, 4><<<grid, 512, SMEM_BYTES, s>>>(p);                \
    else gemm_f64_dmma<BKM, V, L, 2><<<grid, 256, SMEM_BYTES, s>>>(p);                   \
  } while (0)
  if (bk) {
    if (vec2) { if (last) GEMM_GO(true, 2, true); else GEMM_GO(true, 2, false); }
    else { if (last) GEMM_GO(true, 1, true); else GEMM_GO(true, 1, false); }
  } else {
    if (vec2) { if (last) GEMM_GO(false, 2, true); else GEMM_GO(false, 2, false); }
    else { if (last) GEMM_GO(false, 1, true); else GEMM_GO(false, 1, false); }
  }
#undef GEMM_GO
  CUK();
  c->launches++;
  if (S > 1 && !last) {
    reduce_splits<<<grid_for((long)M * N), 256, 0, s>>>(part, S, M, N, C, ldc, sym ? 1 : 0, st);
    CUK();
    c->launches++;
  }
}

// gram of the factor whose columns are the rows of A (r×K, K contiguous) → G (r×r, symmetric).
void gram_launch(enmf_gpu_ctx* c, cudaStream_t s, int prec, const double* A, long lda, int r, int K, double* G,
                 const DevState* st) {
  if (prec == PREC_EXACT) {
    gemm::gram_exact<<<(r * r + 127) / 128, 128, 0, s>>>(A, lda, r, K, G, st);
    CUK();
    c->launches++;
  } else {
    gemm_launch(c, s, true, A, lda, A, lda, G, r, r, r, K, true, st);
  }
}

// ---- inner solvers ------------------------------------------------------------
int hals_variant() {
  // ENMF_HALS_KERNEL: "" persistent paired-warp kernels (default: sweep_tm with the iterate in
  // tensor memory for 64 < r <= 128, sweep_ws below), "wsp" sweep_ws for every r, "ws" one launch
  // per sweep, "fma" CUDA-core kernel.  Retired variants, the timing-experiment builds and their
  // measurements: profiles/r01_sweep_variants.md (the experiment builds are not in the product).
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("ENMF_HALS_KERNEL");
    const std::string s = e ? e : "";
    v = s == "fma" ? 1 : s == "ws" ? 50 : s == "wsp" ? 55 : 54;
  }
  return v;
}

// Tiles (8 columns) per CTA the sweep grid aims for (capped at one CTA per SM).  2 measured
// best from N = 200 to 8192 columns (tools/sweep_grid.sh, profiles/r01_sweep_grid.txt): a
// rank's 4096 columns when C5 is sharded over 8 GPUs sweep in 17.4 µs on 148 CTAs vs 30.0 µs
// on 32 (the previous 16 tiles per CTA); C5 itself fills every SM either way.
// ENMF_SWEEP_TPC overrides (timing experiments).
long sweep_tiles_per_cta() {
  static long v = [] {
    const char* e = std::getenv("ENMF_SWEEP_TPC");
    return e ? std::max(1L, std::atol(e)) : 2L;
  }();
  return v;
}

template <int R_>
void launch_sweep_tf32(enmf_gpu_ctx* c, cudaStream_t s, const hals::Args& a) {
  const long ntiles = ((long)a.N + 7) / 8;
  const unsigned grid = (unsigned)std::max(1L, std::min<long>(c->sms, (ntiles + 15) / 16));
  static bool attr = false;
  if (!attr) {
    CU(cudaFuncSetAttribute((const void*)hals::sweep_tf32<R_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            hals::tf_smem_bytes<R_>()));
    attr = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = hals::tf_smem_bytes<R_>();
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CU(cudaLaunchKernelEx(&lc, hals::sweep_tf32<R_>, a, ntiles));
}

// TF32 variant, r <= 128: right-looking sweeps with the residual in tensor memory and
// tcgen05 rank-8 updates (hals_rl.cuh) when every CTA's columns fit its two 128-column tiles;
// ENMF_TF32_SWEEP=mma keeps the mma.sync left-looking kernel (A/B)
bool sweep_rl_fits(const enmf_gpu_ctx* c, const hals::Args& a) {
  static const bool off = [] {
    const char* e = std::getenv("ENMF_TF32_SWEEP");
    return e && std::strcmp(e, "mma") == 0;
  }();
  // (below ~256 columns the per-solve staging outweighs the faster sweeps: 200×200 r = 20 runs 11%
  // faster on the mma.sync kernel, 10304×400 r = 40 23% slower, tools/tf32_small.py)
  return !off && a.r <= 128 && a.N >= 256 && (long)a.N <= 256L * c->sms;
}

void launch_sweep_rl(enmf_gpu_ctx* c, cudaStream_t s, const hals::Args& a) {
  const unsigned grid = (unsigned)std::max(1L, std::min<long>(c->sms, ((long)a.N + 127) / 128));
  static bool attr = false;
  if (!attr) {
    CU(cudaFuncSetAttribute((const void*)hals::sweep_rl<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            hals::rl_smem_bytes()));
    attr = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(288);   // eight compute warps + the decision warp
  lc.dynamicSmemBytes = hals::rl_smem_bytes();
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CU(cudaLaunchKernelEx(&lc, hals::sweep_rl<128>, a));
}

template <int R_, bool PERSIST = false>
void launch_sweep_ws(enmf_gpu_ctx* c, cudaStream_t s, const hals::Args& a) {
  const long ntiles = ((long)a.N + 7) / 8;
  const long tpc = sweep_tiles_per_cta();
  const unsigned grid = (unsigned)std::max(1L, std::min<long>(c->sms, (ntiles + tpc - 1) / tpc));
  if (PERSIST) {
    // every CTA must be resident for the grid-wide decision between sweeps
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(256);
    lc.dynamicSmemBytes = hals::ws_smem_bytes<R_>();
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CU(cudaLaunchKernelEx(&lc, hals::sweep_ws<R_, true>, a, ntiles));
    return;
  }
  hals::sweep_ws<R_><<<grid, 256, hals::ws_smem_bytes<R_>(), s>>>(a, ntiles);
}

// Persistent TMEM-resident sweep (hals_tm.cuh): 4 column tiles per CTA at least, so small N
// still spreads over the SMs; one CTA per SM (cooperative) for the grid-wide decision.
template <int R_>
void launch_sweep_tm(enmf_gpu_ctx* c, cudaStream_t s, const hals::Args& a) {
  const long ntiles = ((long)a.N + 7) / 8;
  const unsigned grid = (unsigned)std::max(1L, std::min<long>(c->sms, (ntiles + 3) / 4));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = hals::tm_smem_bytes<R_>();
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CU(cudaLaunchKernelEx(&lc, hals::sweep_tm<R_>, a, ntiles));
}


// The persistent sweep kernel runs a whole inner solve in one launch.
bool hals_persistent(int prec, int r) {
  return prec != PREC_EXACT && r <= 128 && (hals_variant() == 54 || hals_variant() == 55);
}

void hals_body(enmf_gpu_ctx* c, cudaStream_t s, const hals::Args& a, int prec) {
  const int r = a.r;
  if (prec == PREC_EXACT || r > 128) {
    hals::sweep_exact<<<(a.N + hals::NT - 1) / hals::NT, hals::NT, 0, s>>>(a);
    CUK();
    hals::gain_exact<<<1, hals::NT, 0, s>>>(a);
    CUK();
    c->launches += 2;
    return;
  }
  const int v = hals_variant();
  if (prec == PREC_TF32 && (v == 54 || v == 55)) {  // TF32 variant: block products on the TF32 tensor cores
    if (sweep_rl_fits(c, a)) launch_sweep_rl(c, s, a);
    else if (r <= 32) launch_sweep_tf32<32>(c, s, a);
    else if (r <= 64) launch_sweep_tf32<64>(c, s, a);
    else launch_sweep_tf32<128>(c, s, a);
  } else if (v == 1) {
#define SW(S_, T_)                                                                          \
  hals::sweep_fast<S_, T_><<<(a.N + hals::NT / T_ - 1) / (hals::NT / T_), hals::NT,          \
                             hals::smem_bytes<S_, T_>(), s>>>(a)
    if (r <= 16) SW(16, 1);
    else if (r <= 32) SW(32, 1);
    else if (r <= 64) SW(32, 2);
    else SW(32, 4);
#undef SW
  } else if (v == 50) {                 // one launch per sweep
    if (r <= 32) launch_sweep_ws<32>(c, s, a);
    else if (r <= 64) launch_sweep_ws<64>(c, s, a);
    else launch_sweep_ws<128>(c, s, a);
  } else {                              // default: persistent, one launch per inner solve
    if (r <= 32) launch_sweep_ws<32, true>(c, s, a);
    else if (r <= 64) launch_sweep_ws<64, true>(c, s, a);
    else if (v == 55) launch_sweep_ws<128, true>(c, s, a);
    else launch_sweep_tm<128>(c, s, a);
  }
  CUK();
  c->launches++;
}

// dv/dscratch/Ntotal: multi-GPU (global max|C|, exchange count and NaN flag across ranks).
// fast: the lane-parallel solver (FP64 product mode, r <= 32); otherwise the bitwise-faithful one
// (fp64_exact, r > 32, and the kernel-level enmf_gpu_active_set_solve).  ENMF_BPP=exact forces the
// latter everywhere.
void bpp_launch(enmf_gpu_ctx* c, cudaStream_t s, const bpp::Args& a, const dist::View* dv = nullptr,
                double* dscratch = nullptr, long Ntotal = 0, bool fast = false) {
  const int r = a.r;
  static const bool force_exact = [] {
    const char* e = std::getenv("ENMF_BPP");
    return e && std::string(e) == "exact";
  }();
  bpp::absmax<<<1, 256, 0, s>>>(a.C, a.ld, r, a.N, const_cast<double*>(a.cmax), a.st, dv);
  CUK();
  if (fast && !force_exact && r <= 32) {
    bpp::solve_fast<8><<<(a.N + 7) / 8, 256, bpp::fast_smem_bytes<8>(), s>>>(a);
  } else if (r <= 32) {
    bpp::solve<32, 8><<<(a.N + 7) / 8, 256, bpp::smem_bytes<32, 8>(), s>>>(a);
  } else if (r <= 64) {
    bpp::solve<64, 4><<<(a.N + 3) / 4, 128, bpp::smem_bytes<64, 4>(), s>>>(a);
  } else {                               // 64 < r <= 128: two-word masks, one warp per block
    bpp::solve<128, 1><<<a.N, 32, bpp::smem_bytes<128, 1>(), s>>>(a);
  }
  CUK();
  if (dv) {
    dist::bpp_check_dist<<<1, 32, 0, s>>>(dv, a.st, a.side, r, Ntotal, a.exchanges, a.rounds, a.nonfinite, dscratch);
  } else {
    bpp::check<<<1, 1, 0, s>>>(a.st, a.side, r, a.N, a.exchanges, a.rounds, a.nonfinite);
  }
  CUK();
  c->launches += 3;
}

// Captures `body(stream)` as the body of a conditional WHILE node appended to
// the graph being captured on `s`.

// driver.inc — run/step control flow (included by engine.cu).
//
// Session = one enmf::run (engine.hpp:447-521):
//   begin : validation (engine.hpp:450-459), upload, ||X||^2, e(0) (:487-503),
//           capture of ONE outer iteration (engine.hpp:309-440) as a CUDA graph
//   step  : launch the graph `count` times (asynchronous, no host round trip)
//   sync  : wait, read the IterationRecords, map device error codes
//   end   : return the accepted factors (RunRecord::factors, :518-520)

// Captures `body(stream)` as the body of a conditional WHILE node appended to
// the graph being captured on `s`.
template <class F>
void capture_while(enmf_gpu_ctx* c, cudaStream_t s, cudaGraphConditionalHandle h, F&& body) {
  cudaStreamCaptureStatus status;
  cudaGraph_t graph;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CU(cudaStreamGetCaptureInfo(s, &status, nullptr, &graph, &deps, &ndeps));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CU(cudaGraphAddNode(&node, graph, deps, ndeps, &np));
  CU(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t bodyg = np.conditional.phGraph_out[0];
  CU(cudaStreamBeginCaptureToGraph(c->body_stream, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  body(c->body_stream);
  cudaGraph_t out;
  CU(cudaStreamEndCapture(c->body_stream, &out));
}

struct Plan {
  int m, n, r;
  int prec;
  int inner_h, inner_w, hp, extrap, literal;
  int max_sweeps_h, max_sweeps_w;
  double stall;
  uint64_t reinit_seed;
};

void validate_cfg(const enmf_gpu_config* c) {
  // SolverConfig::validate (engine.hpp:175-199) with BetaSchedule::validate (:71-81)
  auto bad = [](const char* m) { throw Fail{ENMF_INVALID_ARGUMENT, m}; };
  if (c->hp != 1 && c->hp != 2 && c->hp != 3) bad("SolverConfig: hp must be 1, 2 or 3");
  if (!(c->beta0 >= 0.0) || !(c->beta0 < 1.0)) bad("SolverConfig: beta0 must lie in [0, 1)");
  if (c->extrapolation_enabled && c->beta0 > 0.0) {
    if (!(1.0 < c->gamma_bar) || !(c->gamma_bar < c->gamma) || !(c->gamma < c->eta))
      bad("BetaSchedule: need 1 < gamma_bar < gamma < eta");
  }
  if (!(c->max_seconds > 0.0)) bad("SolverConfig: max_seconds must be > 0");
  if (!(c->inner_sweep_ratio > 0.0)) bad("SolverConfig: inner_sweep_ratio must be > 0");
  if (!(c->inner_stall_fraction > 0.0) || c->inner_stall_fraction >= 1.0)
    bad("SolverConfig: inner_stall_fraction must lie in (0, 1)");
  if ((c->inner_h != ENMF_INNER_EXACT && c->inner_h != ENMF_INNER_HALS) ||
      (c->inner_w != ENMF_INNER_EXACT && c->inner_w != ENMF_INNER_HALS))
    bad("SolverConfig: inner solver must be exact or hals");
  if (c->timing != ENMF_TIMING_WALL && c->timing != ENMF_TIMING_NONE) bad("SolverConfig: bad timing mode");
  if (c->precision != PREC_FAST && c->precision != PREC_EXACT && c->precision != PREC_TF32)
    bad("SolverConfig: unsupported precision");
}

// InnerLoopPolicy::derive (nnls.hpp:79-87) via detail::inner_policy (engine.hpp:250-263)
int derive_sweeps(const enmf_gpu_config* cfg, double setup_flops, size_t rhs, size_t r) {
  if (cfg->inner_max_sweeps) return (int)std::min<uint64_t>(cfg->inner_max_sweeps, 1u << 30);
  const double sweep = (double)rhs * (double)r * (double)r;
  const double rho = sweep > 0.0 ? setup_flops / sweep : 0.0;
  const double v = std::floor(cfg->inner_sweep_ratio * rho);
  return (int)std::min<double>(1.0 + v, (double)(1 << 30));
}

void ensure_buffers(enmf_gpu_ctx* c, size_t m, size_t n, size_t r) {
  const size_t wsz = m * r, hsz = r * n;
  c->WT.ensure(wsz); c->WyT.ensure(wsz); c->WnT.ensure(wsz);
  c->H.ensure(hsz); c->Hy.ensure(hsz); c->Hn.ensure(hsz);
  c->CH.ensure(hsz); c->P.ensure(wsz); c->Plit.ensure(wsz);
  c->GH.ensure(r * r); c->GW.ensure(r * r); c->GWn.ensure(r * r); c->Glit.ensure(r * r);
  c->scratch.ensure(std::max(wsz, hsz));
  const size_t gp = (size_t)std::max(m, n) + 1024;
  c->gain_part.ensure(gp * 2);
  c->part_nf.ensure(gp * 2);
  c->ddpart.ensure(2 * 4096);
  c->dd.ensure(8);
  c->bpp_exch.ensure(2); c->bpp_rounds.ensure(2); c->bpp_nf.ensure(2); c->cmax.ensure(2);
  c->st.ensure(1);
  c->flags.ensure(4);
}

// Products for the error of (W from rows of WTsrc, T): dot = <W, X Tᵀ>, GWn = gram(W).
void enqueue_error_terms(enmf_gpu_ctx* c, cudaStream_t s, const Plan& pl, const double* WTsrc, const double* Pm,
                         DevState* st, int m_loc = -1, const DistHost* D = nullptr) {
  if (m_loc < 0) m_loc = pl.m;
  const long wsz = (long)m_loc * pl.r;
  gram_launch(c, s, pl.prec, WTsrc, m_loc, pl.r, m_loc, c->GWn.p, st);
  if (pl.prec == PREC_EXACT) {
    misc::neumaier_exact<<<1, 32, 0, s>>>(WTsrc, Pm, wsz, 1, pl.r, m_loc, c->dd.p, st);
    CUK();
    c->launches++;
  } else {
    const int nb = (int)std::min<long>(4096, std::max<long>(1, (wsz + 2047) / 2048));
    misc::dd_partial<<<nb, misc::NT, 0, s>>>(WTsrc, Pm, wsz, c->ddpart.p, c->ddpart.p + 4096, st);
    CUK();
    misc::dd_final<<<1, misc::NT, 0, s>>>(c->ddpart.p, c->ddpart.p + 4096, nb, c->dd.p, st);
    CUK();
    c->launches += 2;
  }
  if (D) {  // <W_n, X Tᵀ> and gram(W_n) are sums over the row shards
    dist::allreduce_inplace<<<1, 256, 0, s>>>(D->dview, c->GWn.p, pl.r * pl.r, st);
    dist::allreduce_inplace<<<1, 256, 0, s>>>(D->dview, c->dd.p, 2, st);
    CUK();
    c->launches += 2;
  }
}

// How the data-dependent sweep loop is driven.
enum InnerMode { INNER_CAPTURE = 0, INNER_HOSTLOOP = 1 };

struct Prof {
  cudaEvent_t ev[12];
  double hals_ms[2];
  int hals_sweeps[2];
};

void mark(enmf_gpu_ctx* c, cudaStream_t s, Prof* p, int phase) {
  (void)c;
  if (p) CU(cudaEventRecord(p->ev[phase], s));
}

// CSR products (sparse.cuh): the r-major factor is transposed into the row-major
// scratch, then gathered once per stored entry in the reference's order.
void sparse_gather(enmf_gpu_ctx* c, cudaStream_t s, bool exact, const long long* ptr, const int* idx,
                   const double* val, long lines, const double* Frm, int r, double* out, const DevState* st,
                   const enmf_gpu_ctx::Chunks* ch = nullptr) {
  if (!exact && r <= 32 && ch && ch->n > 0) {
    c->chunk_part.ensure((size_t)std::max(1, ch->nslots) * 32);
    const unsigned grid = (unsigned)std::min<long>(((long)ch->n + 7) / 8, (long)c->sms * 16);
    sparse::gather_chunks<<<grid, 256, 0, s>>>(ch->line.p, ch->beg.p, ch->end.p, ch->slot.p, ch->n, idx, val, Frm, r,
                                               out, lines, c->chunk_part.p, st);
    CUK();
    c->launches++;
    if (ch->nmulti > 0) {
      sparse::combine_chunks<<<(unsigned)std::max(1L, std::min<long>(((long)ch->nmulti * r + 255) / 256, 1024)), 256, 0,
                               s>>>(ch->mline.p, ch->mfirst.p, ch->mcount.p, ch->nmulti, c->chunk_part.p, r, out, lines,
                                    st);
      CUK();
      c->launches++;
    }
    return;
  }
  const long warps = std::max<long>(1, lines);
  const unsigned grid = (unsigned)std::min<long>((warps + 7) / 8, (long)c->sms * 16);
  if (exact) sparse::gather_lines<true><<<grid, 256, 0, s>>>(ptr, idx, val, Frm, (int)lines, r, out, lines, st);
  else if (r <= 32) sparse::gather_lines_par<<<grid, 256, 0, s>>>(ptr, idx, val, Frm, (int)lines, r, out, lines, st);
  else sparse::gather_lines<false><<<grid, 256, 0, s>>>(ptr, idx, val, Frm, (int)lines, r, out, lines, st);
  CUK();
  c->launches++;
}

// Chunk table of a compressed line structure (CSR rows or CSC columns): lines longer than
// `chunk` entries are split (host, once per load).
void build_chunks(enmf_gpu_ctx::Chunks& ch, const std::vector<long long>& ptr, long chunk) {
  std::vector<int> line, slot, mline, mfirst, mcount;
  std::vector<long long> beg, end;
  int nslots = 0;
  const long lines = (long)ptr.size() - 1;
  for (long i = 0; i < lines; ++i) {
    const long long b = ptr[i], e = ptr[i + 1];
    const long long len = e - b;
    const long long nc = std::max<long long>(1, (len + chunk - 1) / chunk);
    if (nc > 1) {
      mline.push_back((int)i);
      mfirst.push_back(nslots);
      mcount.push_back((int)nc);
    }
    for (long long q = 0; q < nc; ++q) {
      line.push_back((int)i);
      beg.push_back(b + q * chunk);
      end.push_back(std::min(e, b + (q + 1) * chunk));
      slot.push_back(nc > 1 ? nslots++ : -1);
    }
  }
  ch.n = (int)line.size();
  ch.nmulti = (int)mline.size();
  ch.nslots = nslots;
  auto up_i = [](DBuf<int>& d, const std::vector<int>& h) {
    d.ensure(std::max<size_t>(1, h.size()));
    if (!h.empty()) CU(cudaMemcpy(d.p, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice));
  };
  auto up_l = [](DBuf<long long>& d, const std::vector<long long>& h) {
    d.ensure(std::max<size_t>(1, h.size()));
    if (!h.empty()) CU(cudaMemcpy(d.p, h.data(), h.size() * sizeof(long long), cudaMemcpyHostToDevice));
  };
  up_i(ch.line, line); up_i(ch.slot, slot); up_i(ch.mline, mline); up_i(ch.mfirst, mfirst); up_i(ch.mcount, mcount);
  up_l(ch.beg, beg); up_l(ch.end, end);
}

void transpose_launch(enmf_gpu_ctx* c, cudaStream_t s, const double* in, double* out, long rows, long cols) {
  dim3 tb(32, 8), tg((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  misc::transpose<<<tg, tb, 0, s>>>(in, out, (int)rows, (int)cols);
  CUK();
  c->launches++;
}

// (X·Tᵀ)ᵀ (r×m) for CSR X, T r×n  (linalg.hpp:127-146)
void sparse_xht(enmf_gpu_ctx* c, cudaStream_t s, bool exact, const double* Tm, int r, double* out,
                const DevState* st) {
  c->rowmaj.ensure(std::max(c->m, c->n) * (size_t)r);
  transpose_launch(c, s, Tm, c->rowmaj.p, r, (long)c->n);
  sparse_gather(c, s, exact, c->csr_ptr.p, c->csr_idx.p, c->csr_val.p, (long)c->m, c->rowmaj.p, r, out, st, &c->ch_csr);
}

// W_yᵀX (r×n) for CSR X (through the CSC copy), W_yᵀ r×m  (linalg.hpp:86-104)
void sparse_wx(enmf_gpu_ctx* c, cudaStream_t s, bool exact, const double* WyT, int r, double* out,
               const DevState* st) {
  c->rowmaj.ensure(std::max(c->m, c->n) * (size_t)r);
  transpose_launch(c, s, WyT, c->rowmaj.p, r, (long)c->m);
  sparse_gather(c, s, exact, c->csc_ptr.p, c->csc_idx.p, c->csc_val.p, (long)c->n, c->rowmaj.p, r, out, st, &c->ch_csc);
}

// ---- FP64 cross products on INT8 tensor cores (ozaki.cuh) ----------------------
// int8 × int8 → int32 digit GEMMs through cuBLASLt (plain library GEMMs); the
// splitting and the FP64 recombination are ours.
// ---- INT8-digit products on the tcgen05 kernels (ozk.cuh) ---------------------------
constexpr int kOzkBN = 128;

// Work split of one digit product (K contracted, N output columns, R factor rows): chunks per
// K unit (≤ 256, so the level sums stay exact in int32) chosen to give ≥ 2 units per SM.
struct OzkPlan { int nkc, unit_chunks, nkq, nmb, ntn; };
OzkPlan ozk_plan(const enmf_gpu_ctx* c, long K, long N, long R) {
  OzkPlan p;
  p.nkc = (int)((K + ozk::KC - 1) / ozk::KC);
  p.nmb = (int)((R + 127) / 128);
  p.ntn = (int)((N + kOzkBN - 1) / kOzkBN);
  const long want = (long)p.nkc * p.ntn * p.nmb / (4L * (c->sms / 2));   // ≥ ~4 units per cluster
  p.unit_chunks = (int)std::max(1L, std::min<long>(ozk::UNIT_CHUNKS, want));
  p.nkq = (p.nkc + p.unit_chunks - 1) / p.unit_chunks;
  return p;
}

// Use the INT8-digit products for the dense FP64 path when the problem is large enough to pay
// the one-time digit cut of X (any shape: TMA fills the ragged tile edges with zero digits).
bool ozaki_enabled(const enmf_gpu_ctx* c, int prec, bool dist) {
  static int env = -1;
  if (env < 0) {
    const char* e = std::getenv("ENMF_CROSS");
    env = (e && std::string(e) == "dmma") ? 0 : 1;
  }
  return env == 1 && prec == PREC_FAST && !c->sparse && (c->x || dist) &&
         (double)c->m * (double)c->n >= (double)(1 << 24);
}

// digits of an X operand (rows × cols, row-major): once per loaded X (outside the iteration graph).
// by_row: one exponent per X row (the operand of T·Xᵀ, whose output columns are X's rows);
// otherwise one per X column (W_yᵀX) — so the product's precision follows each output
// column's own scale, not X's global maximum.  Written in ozk's chunked K-major layout: the
// digit operand has N = rows (by_row) or cols rows, each contracted over the other index.
void ozaki_prepare_x(enmf_gpu_ctx* c, cudaStream_t s, enmf_gpu_ctx::XDig& xd, const double* x, long rows,
                     long cols, bool by_row) {
  if (xd.ready && xd.src == x && xd.rows == rows && xd.cols == cols && xd.by_row == by_row) return;
  const long N = by_row ? rows : cols, K = by_row ? cols : rows;
  const long Kp = (K + ozk::KC - 1) / ozk::KC * ozk::KC, Np = (N + ozk::TROWS - 1) / ozk::TROWS * ozk::TROWS;
  xd.d.ensure((size_t)ozk::SMAX * Kp * Np);
  CU(cudaMemsetAsync(xd.d.p, 0, (size_t)ozk::SMAX * Kp * Np, s));   // padding rows stay zero digits
  xd.e.ensure((size_t)N);
  // digit levels: the neglected terms of level S scale with K·max|a|·max|b| / |sum a·b|; the
  // factor rows inherit X's scales along the contracted index, so X's own max/mean ratio
  // along it stands in for both operands: 6 levels up to 2.5, 7 up to 16, beyond that the
  // product stays on the FP64 DMMA GEMM (levels = 0)
  constexpr int kChunks = 64;
  c->opart.ensure(1 + (by_row ? 0 : 2 * (size_t)kChunks * cols));
  CU(cudaMemsetAsync(c->opart.p, 0, sizeof(double), s));
  auto* rb = reinterpret_cast<unsigned long long*>(c->opart.p);
  if (by_row) {
    ozaki::row_stats<<<(unsigned)rows, 256, 0, s>>>(x, cols, cols, xd.e.p, rb);
  } else {
    double* pm = c->opart.p + 1;
    double* ps = pm + (size_t)kChunks * cols;
    ozaki::col_stats_part<<<dim3((unsigned)((cols + 255) / 256), kChunks), 256, 0, s>>>(x, rows, cols, cols, kChunks,
                                                                                         pm, ps);
    ozaki::col_stats_final<<<(unsigned)std::min<long>((cols + 255) / 256, (long)c->sms * 8), 256, 0, s>>>(
        pm, ps, rows, cols, kChunks, xd.e.p, rb);
  }
  CUK();
  double ratio = 0.0;
  CU(cudaMemcpyAsync(&ratio, c->opart.p, sizeof ratio, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  xd.levels = ratio <= 2.5 ? 6 : ratio <= 16.0 ? 7 : 0;
  c->launches += by_row ? 1 : 2;
  xd.sums.ensure((size_t)ozk::SMAX * N);
  CU(cudaMemsetAsync(xd.sums.p, 0, (size_t)ozk::SMAX * N * sizeof(int), s));
  const long nkc = Kp / ozk::KC;
  const unsigned groups = (unsigned)std::max<long>(1, std::min<long>(nkc, std::max<long>(1, 4L * c->sms * 256 / N)));
  if (by_row)
    ozk::split_rows_chunked<<<dim3((unsigned)((N + 127) / 128), groups), 128, 0, s>>>(x, rows, cols, cols, xd.e.p,
                                                                                     nullptr, xd.d.p, xd.sums.p, nullptr);
  else
    ozk::split_cols_chunked<<<dim3((unsigned)((N + 127) / 128), groups), 128, 0, s>>>(x, rows, cols, cols, xd.e.p,
                                                                                     xd.d.p, xd.sums.p);
  CUK();
  c->launches++;
  xd.N = N;
  xd.K = K;
  xd.by_row = by_row;
  xd.src = x;
  xd.rows = rows;
  xd.cols = cols;
  xd.ready = true;
}

// FP64 partial slices per unit: one per CTA of the pair (ozk::gemm_pair)
int ozk_cluster() { return 2; }

template <int S>
void ozk_launch_pair(enmf_gpu_ctx* c, cudaStream_t s, const int8_t* A, const int8_t* B, const OzkPlan& p, long R, long N,
                     const DevState* st) {
  using Cf = ozk::PairCfg<S>;
  auto kern = ozk::gemm_pair<S>;
  static bool attr = false;
  if (!attr) {
    CU(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
    attr = true;
  }
  ozk::GemmArgs g{A, B, (int)((R + ozk::TROWS - 1) / ozk::TROWS), (int)((N + ozk::TROWS - 1) / ozk::TROWS),
                  (int)R, (int)N, p.nkc, p.unit_chunks, p.nkq, p.nmb, p.ntn, c->ozws.p, st};
  const long items = (long)p.nkq * p.nmb * p.ntn;
  static int maxc = [&] {                 // co-resident CTA pairs (persistent grid, one wave)
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3((unsigned)(c->sms / 2 * 2));
    q.blockDim = dim3(ozk::THREADS);
    q.dynamicSmemBytes = Cf::SMEM;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = 2;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &q) != cudaSuccess || n <= 0) n = c->sms / 2;
    return std::min(n, c->sms / 2);
  }();
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(std::min<long>(items, maxc) * 2));
  lc.blockDim = dim3(ozk::THREADS);
  lc.dynamicSmemBytes = Cf::SMEM;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  CU(cudaLaunchKernelEx(&lc, kern, g));
}

template <int S>
void ozk_launch(enmf_gpu_ctx* c, cudaStream_t s, const int8_t* A, const int8_t* B, const OzkPlan& p, long R, long N,
                const DevState* st) {
  ozk_launch_pair<S>(c, s, A, B, p, R, N, st);
}

// out (r × N, row stride ldo) = A (r × K FP64, row stride lda) · Xdᵀ in FP64 accuracy, Xd = the
// digit operand (N × K).  Returns false (nothing enqueued) when X's dynamic range puts this
// product on the DMMA GEMM instead.
bool ozaki_cross(enmf_gpu_ctx* c, cudaStream_t s, const double* A, long lda, int r, bool tn, double* out, long ldo,
                 const DevState* st, const enmf_gpu_ctx::XDig& xd) {
  (void)tn;
  const int S = xd.levels;
  if (S == 0) return false;
  if (!xd.ready) throw Fail{ENMF_CUDA_ERROR, "internal: X digits not prepared"};
  const long K = xd.K, N = xd.N;
  const OzkPlan p = ozk_plan(c, K, N, r);
  // sized once for every product of this context's shapes: no reallocation between captured launches
  {
    const long mx = (long)std::max(c->m, c->n), mxp = (mx + ozk::KC - 1) / ozk::KC * ozk::KC;
    const size_t an = (size_t)ozk::SMAX * mxp * ((r + ozk::TROWS - 1) / ozk::TROWS * ozk::TROWS);
    if (c->adig.n < an) {                 // tile rows past r stay zero digits (split writes rows < r only)
      c->adig.ensure(an);
      CU(cudaMemsetAsync(c->adig.p, 0, an, s));
    }
    const long dm = c->dist ? (long)c->dist->mp : (long)c->m, dn = c->dist ? (long)c->dist->np : (long)c->n;
    const OzkPlan p1 = ozk_plan(c, (long)c->m, dn, r), p2 = ozk_plan(c, (long)c->n, dm, r);
    c->ozws.ensure((size_t)ozk_cluster() *
                   std::max({(size_t)p1.nkq * r * dn, (size_t)p2.nkq * r * dm, (size_t)p.nkq * r * N}));
  }
  c->aexp.ensure((size_t)r);
  c->asum.ensure((size_t)ozk::SMAX * r);
  c->amax.ensure((size_t)r);
  CU(cudaMemsetAsync(c->amax.p, 0, (size_t)r * sizeof(unsigned long long), s));
  CU(cudaMemsetAsync(c->asum.p, 0, (size_t)ozk::SMAX * r * sizeof(int), s));
  const unsigned kb = (unsigned)std::max<long>(1, std::min<long>((K + 2047) / 2048, 64));
  ozaki::row_absmax<<<dim3(kb, r), 256, 0, s>>>(A, K, lda, c->amax.p, st);
  const long nkc = p.nkc;
  const unsigned groups = (unsigned)std::max<long>(1, std::min<long>(nkc, 4L * c->sms * 128 / std::max(r, 1)));
  ozk::split_rows_chunked<<<dim3((unsigned)((r + 127) / 128), groups), 128, 0, s>>>(A, r, K, lda, c->aexp.p, c->amax.p,
                                                                                   c->adig.p, c->asum.p, st);
  CUK();
  // the factor's box: all S digit tiles at once, or one digit tile per (multicast) load in a cluster
  if (S == 6) ozk_launch<6>(c, s, c->adig.p, xd.d.p, p, r, N, st);
  else ozk_launch<7>(c, s, c->adig.p, xd.d.p, p, r, N, st);
  CUK();
  const dim3 fg((unsigned)std::max<long>(1, std::min<long>((N + 255) / 256, 64)), (unsigned)r);
  if (S == 6)
    ozk::finish<6><<<fg, 256, 0, s>>>(c->ozws.p, p.nkq * ozk_cluster(), r, N, K, c->aexp.p, xd.e.p, c->asum.p, xd.sums.p, out, ldo, st);
  else
    ozk::finish<7><<<fg, 256, 0, s>>>(c->ozws.p, p.nkq * ozk_cluster(), r, N, K, c->aexp.p, xd.e.p, c->asum.p, xd.sums.p, out, ldo, st);
  CUK();
  c->launches += 4;
  return true;
}

// ---- TF32 variant of the cross products (ENMF_PRECISION_TF32) -----------------
// X packed once per load into the TF32 tile images of both products (tf32k.cuh), the factor
// per product; the products on the tcgen05 TF32 kernel (FP32 accumulation); everything else
// (Grams, sweeps, error, decisions) stays FP64.
bool tf32_enabled(const enmf_gpu_ctx* c, int prec, bool dist) {
  return prec == PREC_TF32 && !dist && !c->sparse && c->x;
}

size_t tf32_img_elems(long rows, long K, int RT) {
  return (size_t)((K + tf32k::KE - 1) / tf32k::KE * tf32k::KE) * (size_t)((rows + RT - 1) / RT * RT);
}

void tf32_prepare_x(enmf_gpu_ctx* c, cudaStream_t s) {
  if (c->xf_ready) return;
  const long m = (long)c->m, n = (long)c->n;
  const size_t er = tf32_img_elems(m, n, tf32k::BROWS), ec = tf32_img_elems(n, m, tf32k::BROWS);
  c->xf.ensure(er + ec);                    // [rows image (N = m, K = n) | columns image (N = n, K = m)]
  CU(cudaMemsetAsync(c->xf.p, 0, (er + ec) * sizeof(float), s));
  const unsigned g = (unsigned)std::min<long>((m * n + 255) / 256, (long)c->sms * 64);
  tf32k::pack_rows<<<g, 256, 0, s>>>(c->x, m, n, n, tf32k::BROWS, c->xf.p, nullptr);
  tf32k::pack_cols<<<g, 256, 0, s>>>(c->x, m, n, tf32k::BROWS, c->xf.p + er);
  CUK();
  c->launches += 2;
  c->xf_ready = true;
}

void tf32_cross(enmf_gpu_ctx* c, cudaStream_t s, const double* A, long lda, int r, bool tn, double* out, long ldo,
                const DevState* st) {
  const long m = (long)c->m, n = (long)c->n;
  const long K = tn ? n : m, N = tn ? m : n;
  const float* B = c->xf.p + (tn ? 0 : tf32_img_elems(m, n, tf32k::BROWS));
  const size_t an = tf32_img_elems(r, std::max(m, n), tf32k::AROWS);
  if (c->af.n < an) {                       // padding rows past r stay zero
    c->af.ensure(an);
    CU(cudaMemsetAsync(c->af.p, 0, an * sizeof(float), s));
  }
  tf32k::pack_rows<<<(unsigned)std::min<long>(((long)r * K + 255) / 256, (long)c->sms * 16), 256, 0, s>>>(
      A, r, K, lda, tf32k::AROWS, c->af.p, st);
  CUK();
  tf32k::Args g{};
  g.A = c->af.p; g.B = B;
  g.nta = (r + tf32k::AROWS - 1) / tf32k::AROWS; g.ntb = (int)((N + tf32k::BROWS - 1) / tf32k::BROWS);
  g.R = r; g.N = (int)N; g.nkc = (int)((K + tf32k::KE - 1) / tf32k::KE);
  const long tiles = (long)g.nta * g.ntb;
  g.nks = (int)std::max(1L, std::min<long>(g.nkc, (4L * c->sms + tiles - 1) / tiles));   // ≥ ~4 items per SM
  g.split_chunks = (g.nkc + g.nks - 1) / g.nks;
  g.nks = (g.nkc + g.split_chunks - 1) / g.split_chunks;
  // partials sized once for both products (no reallocation between captured launches)
  {
    const long tl = (long)((std::max(m, n) + tf32k::BROWS - 1) / tf32k::BROWS) * g.nta;
    const long nkcm = (std::max(m, n) + tf32k::KE - 1) / tf32k::KE;
    const long ks = std::min<long>(nkcm, (4L * c->sms + tl - 1) / tl) + 1;
    c->cf.ensure(std::max((size_t)g.nks * r * N, (size_t)ks * r * std::max(m, n)));
  }
  g.part = c->cf.p;
  g.st = st;
  static bool attr = false;
  if (!attr) {
    CU(cudaFuncSetAttribute((const void*)tf32k::gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, tf32k::SMEM));
    attr = true;
  }
  const long items = (long)g.nks * tiles;
  tf32k::gemm<<<(unsigned)std::min<long>(items, c->sms), tf32k::THREADS, tf32k::SMEM, s>>>(g);
  CUK();
  tf32k::finish<<<(unsigned)std::min<long>(((long)r * N + 255) / 256, (long)c->sms * 16), 256, 0, s>>>(
      c->cf.p, g.nks, r, N, out, ldo, st);
  CUK();
  c->launches += 3;
}

// sweep_ws reads the Gram in A-fragment order: arrange it once per inner solve.
void ws_prepare(enmf_gpu_ctx* c, cudaStream_t s, hals::Args& a, int prec, int slot) {
  if (prec == PREC_EXACT || a.r > 128) return;
  constexpr size_t kGf = 128 * 128 + 64 * 64;   // fragments + tails (ws_prep)
  c->Gf.ensure(3 * kGf);
  double* gf = c->Gf.p + slot * kGf;
  if (prec == PREC_TF32 && (hals_variant() == 54 || hals_variant() == 55)) {   // TF32 variant's sweep: m16n8k8 fragments (tf_prep)
    auto* gf4 = reinterpret_cast<float4*>(gf);
    if (a.r <= 32) hals::tf_prep<32><<<8, 256, 0, s>>>(a.G, a.r, gf4, a.st, a.ctl);
    else if (a.r <= 64) hals::tf_prep<64><<<16, 256, 0, s>>>(a.G, a.r, gf4, a.st, a.ctl);
    else hals::tf_prep<128><<<64, 256, 0, s>>>(a.G, a.r, gf4, a.st, a.ctl);
    CUK();
    c->launches++;
    a.Gf = gf;
    return;
  }
  if (hals_variant() != 50 && hals_variant() != 54 && hals_variant() != 55) return;
  if (a.r <= 32) hals::ws_prep<32><<<8, 256, 0, s>>>(a.G, a.r, gf, a.st, a.ctl);
  else if (a.r <= 64) hals::ws_prep<64><<<16, 256, 0, s>>>(a.G, a.r, gf, a.st, a.ctl);
  else if (hals_variant() == 50 || hals_variant() == 55) hals::ws_prep<128><<<64, 256, 0, s>>>(a.G, a.r, gf, a.st, a.ctl);
  else hals::ws_prep<128, true, true><<<64, 256, 0, s>>>(a.G, a.r, gf, a.st, a.ctl);   // sweep_tm: rows / G_kk
  CUK();
  c->launches++;
  a.Gf = gf;
}

void enqueue_inner(enmf_gpu_ctx* c, cudaStream_t s, const Plan& pl, int side, int solver, const double* G,
                   const double* Cm, const double* Hin, double* Hout, int rows_n, int max_sweeps, DevState* st,
                   cudaGraphConditionalHandle cond, int mode, Prof* prof, const DistHost* D = nullptr,
                   long rows_total = 0) {
  if (solver == ENMF_INNER_HALS) {
    hals::Args a{};
    a.G = G; a.C = Cm; a.Hin = Hin; a.H = Hout; a.ld = rows_n; a.r = pl.r; a.N = rows_n;
    a.max_sweeps = max_sweeps; a.stall = pl.stall;
    a.ctl = &st->hals[side];
    a.part = c->gain_part.p + side * (c->gain_part.n / 2);
    a.part_nf = c->part_nf.p + side * (c->part_nf.n / 2);
    a.terms = c->terms.p; a.st = st; a.side = side;
    a.H2 = c->scratch.p;                 // r·max(m, n): unused while the iteration graphs run
    a.cond = (unsigned long long)cond; a.use_cond = mode == INNER_CAPTURE ? 1 : 0;
    a.dv = D ? D->dview : nullptr;
    hals::reset_ctl<<<1, 1, 0, s>>>(a.ctl, st);
    CUK();
    c->launches++;
    ws_prepare(c, s, a, pl.prec, side);
    if (mode == INNER_CAPTURE) {
      if (hals_persistent(pl.prec, pl.r)) {
        a.use_cond = 0;                       // one launch runs every sweep
        hals_body(c, s, a, pl.prec);
      } else {
        capture_while(c, s, cond, [&](cudaStream_t bs) { hals_body(c, bs, a, pl.prec); });
      }
    } else {
      // host-driven: one sweep per launch, flag read back after each (profiling / no-graph path)
      cudaEvent_t e0, e1;
      CU(cudaEventCreate(&e0));
      CU(cudaEventCreate(&e1));
      double ms = 0.0;
      int sweeps = 0;
      for (int i = 0; i < max_sweeps; ++i) {
        CU(cudaEventRecord(e0, s));
        hals_body(c, s, a, pl.prec);
        CU(cudaEventRecord(e1, s));
        HalsCtl hc;
        CU(cudaMemcpyAsync(&hc, a.ctl, sizeof hc, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        float t = 0.f;
        CU(cudaEventElapsedTime(&t, e0, e1));
        ms += t;
        sweeps = hc.sweeps;
        if (!hc.cont) break;
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      if (prof) {
        prof->hals_ms[side] = ms;
        prof->hals_sweeps[side] = sweeps;
      }
    }
  } else {
    bpp::Args a{};
    a.G = G; a.C = Cm; a.H0 = Hin; a.H = Hout; a.ld = rows_n; a.r = pl.r; a.N = rows_n;
    a.cmax = c->cmax.p + side; a.st = st; a.side = side;
    a.exchanges = c->bpp_exch.p + side; a.rounds = c->bpp_rounds.p + side; a.nonfinite = c->bpp_nf.p + side;
    const bool fast = pl.prec != PREC_EXACT;
    if (D) bpp_launch(c, s, a, D->dview, D->scratch, rows_total, fast);
    else bpp_launch(c, s, a, nullptr, nullptr, 0, fast);
  }
}

// Where the data of an iteration lives: the whole problem (single GPU) or this
// rank's shards plus the full factor replicas (multi-GPU).
struct Layout {
  int m_loc, n_loc;               // rows of W / columns of H held here
  long row0, col0;
  const double* xcb; long ld_cb;  // X[:, J]  (m × n_loc)  for W_yᵀX
  const double* xrb; long ld_rb;  // X[I, :]  (m_loc × n)  for X·Tᵀ
  double* wyfull;                 // W_yᵀ replica (r × m), own rank
  double* tfull;                  // T replica (r × n), own rank
  const DistHost* D;              // null on a single GPU
};

Layout make_layout(enmf_gpu_ctx* c, const Plan& pl) {
  Layout L{};
  const DistHost* D = (c->dist && c->dist->ready) ? c->dist : nullptr;
  L.D = D;
  if (!D) {
    L.m_loc = pl.m; L.n_loc = pl.n; L.row0 = 0; L.col0 = 0;
    L.xcb = c->x; L.ld_cb = pl.n; L.xrb = c->x; L.ld_rb = pl.n;
    L.wyfull = c->WyT.p; L.tfull = nullptr;
  } else {
    L.m_loc = (int)D->mp; L.n_loc = (int)D->np; L.row0 = (long)D->row0; L.col0 = (long)D->col0;
    L.xcb = D->xc; L.ld_cb = (long)D->np; L.xrb = D->xr; L.ld_rb = pl.n;
    L.wyfull = D->wfull(D->rank); L.tfull = D->tfull(D->rank);
  }
  return L;
}

// Multi-GPU helpers (no-ops on one GPU).
void dist_allreduce(enmf_gpu_ctx* c, cudaStream_t s, const Layout& L, double* buf, int count, DevState* st) {
  if (!L.D) return;
  dist::allreduce_inplace<<<1, 256, 0, s>>>(L.D->dview, buf, count, st);
  CUK();
  c->launches++;
}
// which: 0 = W_yᵀ replica (columns I = [row0, row0+m_loc) of r×m), 1 = T replica (columns J of r×n)
void dist_gather(enmf_gpu_ctx* c, cudaStream_t s, const Layout& L, const double* local, int r, int which,
                 const Plan& pl, DevState* st) {
  if (!L.D) return;
  const long cnt = which == 0 ? L.m_loc : L.n_loc;
  const long off = which == 0 ? L.row0 : L.col0;
  const long full = which == 0 ? pl.m : pl.n;
  dist::scatter_shard_k<<<grid_for((long)r * cnt), 256, 0, s>>>(L.D->dview, local, r, cnt, off, full, which, st);
  dist::barrier_k<<<1, 32, 0, s>>>(L.D->dview, st);
  CUK();
  c->launches += 2;
}

// One outer iteration, step() of engine.hpp:309-440.
void enqueue_iteration(enmf_gpu_ctx* c, cudaStream_t s, const Plan& pl, cudaGraphConditionalHandle ch,
                       cudaGraphConditionalHandle cw, int mode, Prof* prof) {
  DevState* st = c->st.p;
  const Layout L = make_layout(c, pl);
  const DistHost* D = L.D;
  const int m = pl.m, n = pl.n, r = pl.r;
  const int ml = L.m_loc, nl = L.n_loc;
  const long wsz = (long)ml * r, hsz = (long)r * nl;
  mark(c, s, prof, 0);
  misc::iter_begin<<<1, 1, 0, s>>>(st);
  CUK();
  c->launches++;

  auto fixup = [&](double* A, int cnt, long off, long full, int which, double* G, int side) {
    if (D) {
      dist::reinit_fixup_dist<<<1, 256, 0, s>>>(D->dview, A, r, cnt, off, full, which, G, pl.reinit_seed, side, st);
    } else {
      misc::reinit_fixup<<<1, misc::NT, 0, s>>>(A, cnt, r, cnt, G, pl.reinit_seed, side, st);
    }
    CUK();
    c->launches++;
  };

  // ---- H update (engine.hpp:323-337) ----
  // (multi-GPU: the W_yᵀ replica was assembled at the end of the previous iteration / in begin)
  gram_launch(c, s, pl.prec, c->WyT.p, ml, r, ml, c->GH.p, st);
  dist_allreduce(c, s, L, c->GH.p, r * r, st);
  fixup(c->WyT.p, ml, L.row0, m, 0, c->GH.p, 0);
  mark(c, s, prof, 1);
  if (c->sparse) {
    sparse_wx(c, s, pl.prec == PREC_EXACT, c->WyT.p, r, c->CH.p, st);
  } else if (tf32_enabled(c, pl.prec, D != nullptr)) {
    tf32_cross(c, s, c->WyT.p, m, r, false, c->CH.p, n, st);
  } else if (ozaki_enabled(c, pl.prec, D != nullptr) &&
             ozaki_cross(c, s, L.wyfull, m, r, false, c->CH.p, nl, st, D ? c->xd_cols : c->xd_x)) {
    // on the INT8 tensor cores
  } else if (pl.prec == PREC_EXACT) {
    gemm::cross_wx_exact<<<grid_for(hsz, 128, 1 << 30), 128, 0, s>>>(c->WyT.p, c->x, m, n, r, c->CH.p, st);
    CUK();
    c->launches++;
  } else {
    gemm_launch(c, s, false, L.wyfull, m, L.xcb, L.ld_cb, c->CH.p, nl, r, nl, m, false, st);
  }
  mark(c, s, prof, 2);
  enqueue_inner(c, s, pl, 0, pl.inner_h, c->GH.p, c->CH.p, c->Hy.p, c->Hn.p, nl, pl.max_sweeps_h, st, ch, mode, prof,
                D, n);
  mark(c, s, prof, 3);

  // ---- early H extrapolation (engine.hpp:340-347) ----
  if (pl.hp >= 2) {
    if (pl.extrap) misc::extrap<<<grid_for(hsz), 256, 0, s>>>(c->Hn.p, c->H.p, c->Hy.p, hsz, pl.hp == 3, st);
    else misc::copy<<<grid_for(hsz), 256, 0, s>>>(c->Hn.p, c->Hy.p, hsz, st);
    CUK();
    c->launches++;
  }
  const bool target_hy = pl.hp >= 2 || (pl.literal && pl.extrap);
  double* T = target_hy ? c->Hy.p : c->Hn.p;
  mark(c, s, prof, 4);

  // ---- W update (engine.hpp:353-383) ----
  dist_gather(c, s, L, T, r, 1, pl, st);                 // T replica for X·Tᵀ
  gram_launch(c, s, pl.prec, T, nl, r, nl, c->GW.p, st);
  dist_allreduce(c, s, L, c->GW.p, r * r, st);
  fixup(T, nl, L.col0, n, 1, c->GW.p, 1);
  mark(c, s, prof, 5);
  auto cross_xht = [&](const double* Tm, double* out) {
    if (c->sparse) {
      sparse_xht(c, s, pl.prec == PREC_EXACT, Tm, r, out, st);
    } else if (tf32_enabled(c, pl.prec, D != nullptr)) {
      tf32_cross(c, s, Tm, n, r, true, out, m, st);
    } else if (ozaki_enabled(c, pl.prec, D != nullptr) &&
               ozaki_cross(c, s, D ? L.tfull : Tm, n, r, true, out, ml, st, D ? c->xd_rows : c->xd_xt)) {
      // on the INT8 tensor cores
    } else if (pl.prec == PREC_EXACT) {
      gemm::cross_xht_exact<<<grid_for(wsz, 128, 1 << 30), 128, 0, s>>>(c->x, Tm, m, n, r, out, st);
      CUK();
      c->launches++;
    } else {
      gemm_launch(c, s, true, D ? L.tfull : Tm, n, L.xrb, L.ld_rb, out, ml, r, ml, n, false, st);
    }
  };
  cross_xht(T, c->P.p);
  mark(c, s, prof, 6);
  enqueue_inner(c, s, pl, 1, pl.inner_w, c->GW.p, c->P.p, c->WyT.p, c->WnT.p, ml, pl.max_sweeps_w, st, cw, mode,
                prof, D, m);
  mark(c, s, prof, 7);

  // ---- error (engine.hpp:402-416) ----
  const double* Pe = c->P.p;
  const double* Ge = c->GW.p;
  int mode_h = pl.hp >= 2 ? 0 : 1;
  if (pl.hp == 1 && pl.literal && pl.extrap) {
    misc::extrap<<<grid_for(hsz), 256, 0, s>>>(c->Hn.p, c->H.p, c->Hy.p, hsz, 0, st);
    CUK();
    c->launches++;
    dist_gather(c, s, L, c->Hy.p, r, 1, pl, st);
    gram_launch(c, s, pl.prec, c->Hy.p, nl, r, nl, c->Glit.p, st);
    dist_allreduce(c, s, L, c->Glit.p, r * r, st);
    cross_xht(c->Hy.p, c->Plit.p);
    Pe = c->Plit.p;
    Ge = c->Glit.p;
    mode_h = 2;
  }
  enqueue_error_terms(c, s, pl, c->WnT.p, Pe, st, ml, D);
  mark(c, s, prof, 8);
  misc::decide<<<1, misc::NT, 0, s>>>(st, c->dd.p, c->GWn.p, Ge, r, pl.prec == PREC_EXACT, c->recs.p, 0);
  CUK();
  misc::finalize<<<grid_for(std::max(wsz, hsz)), 256, 0, s>>>(c->WT.p, c->WyT.p, c->WnT.p, wsz, c->H.p, c->Hy.p,
                                                              c->Hn.p, hsz, mode_h, st);
  CUK();
  c->launches += 2;
  dist_gather(c, s, L, c->WyT.p, r, 0, pl, st);          // W_yᵀ replica for the next iteration
  mark(c, s, prof, 9);
}

void set_err(const Fail& f) { g_last_error = f.msg; }

}  // namespace

struct Session {
  Plan pl{};
  bool dev_factors = false;
  size_t m = 0, n = 0, r = 0;
  size_t ml = 0, nl = 0;    // local extents (rows of W, columns of H held here)
  size_t K = 0;             // max_outer_iterations
  size_t launched = 0;      // iterations enqueued so far
  size_t counted = 0;       // iterations whose kernels were added to c->launches
  int static_kernels = 0;   // per-iteration kernels outside the sweep loops
  int kps = 1;              // kernels per HALS sweep
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool failed = false;
};

namespace {

// Host X → device on the copy stream (DenseMatrix data, matrix.hpp:65-66); returns at once for
// pinned memory.  The engine stream joins it in x_join, right before X is first read.
void x_upload_async(enmf_gpu_ctx* c, const double* x, size_t m, size_t n) {
  if (!c->copy_stream) {
    CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&c->x_copied, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->x_checked, cudaEventDisableTiming));
    CU(cudaHostAlloc(reinterpret_cast<void**>(&c->x_bad), sizeof(int), cudaHostAllocDefault));
  }
  if (c->x_state == 2) CU(cudaEventSynchronize(c->x_checked));   // an unread verdict of the previous X: dropped
  c->x_own.ensure(m * n);
  // the previous X may still be read by work queued on the engine stream
  CU(cudaEventRecord(c->x_checked, c->stream));
  CU(cudaStreamWaitEvent(c->copy_stream, c->x_checked, 0));
  CU(cudaMemcpyAsync(c->x_own.p, x, m * n * 8, cudaMemcpyHostToDevice, c->copy_stream));
  CU(cudaEventRecord(c->x_copied, c->copy_stream));
  c->x = c->x_own.p;
  c->x_state = 1;
}

// The engine stream waits for the copy and checks the values (DenseMatrix rejects NaN/Inf,
// matrix.hpp:43-51) on the device; the verdict lands in pinned memory.
void x_join(enmf_gpu_ctx* c) {
  if (c->x_state != 1) return;
  if (!c->x || c->sparse) {               // another data matrix was loaded since
    c->x_state = 0;
    return;
  }
  cudaStream_t s = c->stream;
  CU(cudaStreamWaitEvent(s, c->x_copied, 0));
  c->flags.ensure(4);
  CU(cudaMemsetAsync(c->flags.p + 1, 0, sizeof(int), s));
  misc::check_factor<<<grid_for((long)(c->m * c->n)), 256, 0, s>>>(c->x, (long)(c->m * c->n), c->flags.p + 1, 0);
  CUK();
  c->launches++;
  CU(cudaMemcpyAsync(c->x_bad, c->flags.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaEventRecord(c->x_checked, s));
  c->x_state = 2;
}

// Reads the verdict once it is in (wait: block for it); a non-finite X fails the call like the
// reference's DenseMatrix constructor.
void x_verdict(enmf_gpu_ctx* c, bool wait) {
  if (c->x_state != 2) return;
  if (wait) CU(cudaEventSynchronize(c->x_checked));
  else if (cudaEventQuery(c->x_checked) != cudaSuccess) { (void)cudaGetLastError(); return; }
  c->x_state = 0;
  if (*c->x_bad) {
    c->x = nullptr;
    throw Fail{ENMF_INVALID_ARGUMENT, "DenseMatrix: values must be finite"};
  }
}

void close_session(enmf_gpu_ctx* c) {
  if (!c->sess) return;
  if (c->sess->exec) cudaGraphExecDestroy(c->sess->exec);
  if (c->sess->graph) cudaGraphDestroy(c->sess->graph);
  delete c->sess;
  c->sess = nullptr;
}

// ENMF_TRACE_BEGIN=1: host wall time of begin()'s phases on stderr (synchronizes the stream)
struct BeginTrace {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t;
  explicit BeginTrace(cudaStream_t s_) : on(std::getenv("ENMF_TRACE_BEGIN") != nullptr), s(s_) {
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto u = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[begin] %-24s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(u - t).count());
    t = u;
  }
};

void begin_impl(enmf_gpu_ctx* c, const double* w0, const double* h0, size_t r, bool dev_factors,
                const enmf_gpu_config* cfg) {
  if (!c) throw Fail{ENMF_INVALID_ARGUMENT, "null context"};
  if (!cfg) throw Fail{ENMF_INVALID_ARGUMENT, "null config"};
  CU(cudaSetDevice(c->device));
  close_session(c);
  validate_cfg(cfg);
  const DistHost* D = (c->dist && c->dist->ready) ? c->dist : nullptr;
  if (!D && !c->x && !c->sparse) throw Fail{ENMF_INVALID_ARGUMENT, "run: no data matrix loaded"};
  if (D && c->sparse) throw Fail{ENMF_INVALID_ARGUMENT, "run: the sharded engine takes dense data only"};
  if (D && (!D->xc || !D->xr)) throw Fail{ENMF_INVALID_ARGUMENT, "run: no sharded data loaded"};
  if (D && cfg->precision == PREC_EXACT)
    throw Fail{ENMF_INVALID_ARGUMENT, "the bitwise-faithful precision is single-GPU only"};
  if (D && r != D->r) throw Fail{ENMF_INVALID_ARGUMENT, "run: rank differs from the one the shared buffers were sized for"};
  const size_t m = c->m, n = c->n;
  // local extents: the whole problem on one GPU, this rank's shards otherwise
  const size_t ml = D ? D->mp : m, nl = D ? D->np : n;
  if (r == 0) throw Fail{ENMF_INVALID_ARGUMENT, "DenseMatrix: rows and cols must be >= 1"};
  if (!w0 || !h0) throw Fail{ENMF_INVALID_ARGUMENT, "run: null initial factor"};
  if (m > (size_t)INT32_MAX || n > (size_t)INT32_MAX || r > 4096)
    throw Fail{ENMF_INVALID_ARGUMENT, "run: shape exceeds the device path's limits (m,n < 2^31, r <= 4096)"};
  if ((cfg->inner_h == ENMF_INNER_EXACT || cfg->inner_w == ENMF_INNER_EXACT) && r > bpp::MAXR)
    throw Fail{ENMF_INVALID_ARGUMENT, "active_set_solve on device supports r <= 128"};
  if ((cfg->inner_h == ENMF_INNER_HALS || cfg->inner_w == ENMF_INNER_HALS) && r > 1024)
    throw Fail{ENMF_INVALID_ARGUMENT, "hals_solve on device supports r <= 1024"};
  if (cfg->max_outer_iterations > (1ULL << 24))
    throw Fail{ENMF_INVALID_ARGUMENT, "max_outer_iterations exceeds the record buffer limit (2^24)"};
  const size_t wsz = ml * r, hsz = r * nl;
  cudaStream_t s = c->stream;
  (void)cudaGetLastError();  // drop a stale (non-sticky) error from an earlier failed call
  BeginTrace tr(s);
  set_attrs_once();
  ensure_buffers(c, ml, nl, r);
  presize_splits(c, s, m, n, ml, nl, r);
  tr.mark("buffers");
  if (cfg->precision == PREC_EXACT || r > 128) c->terms.ensure(std::max(wsz, hsz));
  const size_t K = cfg->max_outer_iterations;
  c->recs.ensure(K + 1);

  // validate + upload factors (engine.hpp:451-459)
  if (!dev_factors) {
    // upload first, then the same finite / nonnegative check on the device (one pass over the
    // 2·r·(m+n) values instead of a host loop)
    CU(cudaMemcpyAsync(c->scratch.p, w0, wsz * 8, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(c->H.p, h0, hsz * 8, cudaMemcpyHostToDevice, s));
    CU(cudaMemsetAsync(c->flags.p, 0, sizeof(int), s));
    misc::check_factor<<<grid_for(wsz), 256, 0, s>>>(c->scratch.p, wsz, c->flags.p, 1);
    misc::check_factor<<<grid_for(hsz), 256, 0, s>>>(c->H.p, hsz, c->flags.p, 1);
    CUK();
    c->launches += 2;
    int bad = 0;
    CU(cudaMemcpyAsync(&bad, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (bad) throw Fail{ENMF_INVALID_ARGUMENT, "run: initial factors must be finite and nonnegative"};
  } else {
    CU(cudaMemsetAsync(c->flags.p, 0, sizeof(int), s));
    misc::check_factor<<<grid_for(wsz), 256, 0, s>>>(w0, wsz, c->flags.p, 1);
    misc::check_factor<<<grid_for(hsz), 256, 0, s>>>(h0, hsz, c->flags.p, 1);
    CUK();
    int bad = 0;
    CU(cudaMemcpyAsync(&bad, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (bad) throw Fail{ENMF_INVALID_ARGUMENT, "run: initial factors must be finite and nonnegative"};
    CU(cudaMemcpyAsync(c->scratch.p, w0, wsz * 8, cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(c->H.p, h0, hsz * 8, cudaMemcpyDeviceToDevice, s));
    c->launches += 2;
  }
  {
    dim3 tb(32, 8), tg((unsigned)((r + 31) / 32), (unsigned)((ml + 31) / 32));
    misc::transpose<<<tg, tb, 0, s>>>(c->scratch.p, c->WT.p, (int)ml, (int)r);
    CUK();
    c->launches++;
  }
  CU(cudaMemcpyAsync(c->WyT.p, c->WT.p, wsz * 8, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemcpyAsync(c->Hy.p, c->H.p, hsz * 8, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemsetAsync(c->bpp_exch.p, 0, 2 * sizeof(unsigned long long), s));
  CU(cudaMemsetAsync(c->bpp_rounds.p, 0, 2 * sizeof(int), s));
  CU(cudaMemsetAsync(c->bpp_nf.p, 0, 2 * sizeof(int), s));
  tr.mark("factors");
  x_join(c);                             // a host X still in flight (enmf_gpu_run_dense): first read below

  // run state (engine.hpp:471-481)
  DevState hs;
  std::memset(&hs, 0, sizeof hs);
  hs.beta = cfg->beta0;
  hs.beta_bar = 1.0;
  hs.beta_prev = cfg->beta0;
  hs.gamma = cfg->gamma;
  hs.gamma_bar = cfg->gamma_bar;
  hs.eta = cfg->eta;
  hs.max_seconds = cfg->max_seconds;
  hs.max_iter = K;
  hs.active = 1;
  hs.extrapolation = cfg->extrapolation_enabled ? 1 : 0;
  hs.hp = cfg->hp;
  hs.wall = (cfg->timing == ENMF_TIMING_WALL || std::isfinite(cfg->max_seconds)) ? 1 : 0;
  hs.literal = cfg->literal_hp1_order ? 1 : 0;
  CU(cudaMemcpyAsync(c->st.p, &hs, sizeof hs, cudaMemcpyHostToDevice, s));
  DevState* st = c->st.p;
  misc::run_begin<<<1, 1, 0, s>>>(st);
  CUK();
  c->launches++;

  auto* se = new Session();
  c->sess = se;
  Plan& pl = se->pl;
  pl.m = (int)m; pl.n = (int)n; pl.r = (int)r;
  pl.prec = cfg->precision;
  pl.inner_h = cfg->inner_h; pl.inner_w = cfg->inner_w; pl.hp = cfg->hp;
  pl.extrap = cfg->extrapolation_enabled ? 1 : 0;
  pl.literal = cfg->literal_hp1_order ? 1 : 0;
  // setup_flop_estimate (engine.hpp:242-248): m·n·r dense, nnz·r sparse
  const double setup = c->sparse ? (double)c->nnz * (double)r : (double)m * (double)n * (double)r;
  pl.max_sweeps_h = derive_sweeps(cfg, setup, n, r);
  pl.max_sweeps_w = derive_sweeps(cfg, setup, m, r);
  pl.stall = cfg->inner_stall_fraction;
  pl.reinit_seed = cfg->reinit_seed;
  se->dev_factors = dev_factors;
  se->m = m; se->n = n; se->r = r; se->K = K;
  se->ml = ml; se->nl = nl;
  se->kps = (pl.prec == PREC_EXACT || r > 128) ? 2 : hals_persistent(pl.prec, (int)r) ? 0 : 1;
  const Layout L = make_layout(c, pl);

  // ||X||^2 (linalg.hpp:160-171) and e(0) (engine.hpp:487-503)
  // (CSR: the stored values in storage order, linalg.hpp:167-171)
  const double* xnorm = c->sparse ? c->csr_val.p : D ? D->xr : c->x;   // multi-GPU: the row blocks partition X
  const long xs = c->sparse ? (long)c->nnz : (long)ml * n;
  if (pl.prec == PREC_EXACT) {
    misc::neumaier_exact<<<1, 32, 0, s>>>(xnorm, nullptr, xs, 0, 0, 0, c->dd.p + 2, nullptr);
    c->launches++;
  } else {
    const int nb = (int)std::min<long>(4096, std::max<long>(1, (xs + 4095) / 4096));
    misc::dd_partial<<<nb, misc::NT, 0, s>>>(xnorm, nullptr, xs, c->ddpart.p, c->ddpart.p + 4096, nullptr);
    misc::dd_final<<<1, misc::NT, 0, s>>>(c->ddpart.p, c->ddpart.p + 4096, nb, c->dd.p + 2, nullptr);
    c->launches += 2;
  }
  CUK();
  dist_allreduce(c, s, L, c->dd.p + 2, 2, st);
  misc::set_norm<<<1, 1, 0, s>>>(st, c->dd.p + 2);
  CUK();
  tr.mark("norm");
  gram_launch(c, s, pl.prec, c->H.p, nl, (int)r, (int)nl, c->GW.p, st);
  dist_allreduce(c, s, L, c->GW.p, (int)(r * r), st);
  dist_gather(c, s, L, c->H.p, (int)r, 1, pl, st);       // H0 replica for X·H0ᵀ
  dist_gather(c, s, L, c->WT.p, (int)r, 0, pl, st);      // W0ᵀ replica for iteration 1's W_yᵀX
  if (c->sparse) {
    sparse_xht(c, s, pl.prec == PREC_EXACT, c->H.p, (int)r, c->P.p, st);
  } else if (tf32_enabled(c, pl.prec, D != nullptr)) {
    tf32_prepare_x(c, s);                // once per loaded X (outside the iteration graph)
    tf32_cross(c, s, c->H.p, (long)n, (int)r, true, c->P.p, (long)m, st);
  } else if (ozaki_enabled(c, pl.prec, D != nullptr)) {
    if (D) {                             // once per loaded X (outside the iteration graph)
      ozaki_prepare_x(c, s, c->xd_cols, D->xc, (long)m, (long)D->np, false);
      ozaki_prepare_x(c, s, c->xd_rows, D->xr, (long)D->mp, (long)n, true);
    } else {
      ozaki_prepare_x(c, s, c->xd_x, c->x, (long)m, (long)n, false);
      tr.mark("digits x (cols)");
      ozaki_prepare_x(c, s, c->xd_xt, c->x, (long)m, (long)n, true);
      tr.mark("digits x (rows)");
    }
    if (!ozaki_cross(c, s, D ? L.tfull : c->H.p, (long)n, (int)r, true, c->P.p, (long)ml, st,
                     D ? c->xd_rows : c->xd_xt))
      gemm_launch(c, s, true, D ? L.tfull : c->H.p, n, L.xrb, L.ld_rb, c->P.p, ml, (int)r, (int)ml, (int)n, false,
                  st);
  } else if (pl.prec == PREC_EXACT) {
    gemm::cross_xht_exact<<<grid_for((long)wsz, 128, 1 << 30), 128, 0, s>>>(c->x, c->H.p, (int)m, (int)n, (int)r,
                                                                             c->P.p, st);
    CUK();
    c->launches++;
  } else {
    gemm_launch(c, s, true, D ? L.tfull : c->H.p, n, L.xrb, L.ld_rb, c->P.p, ml, (int)r, (int)ml, (int)n, false, st);
  }
  enqueue_error_terms(c, s, pl, c->WT.p, c->P.p, st, (int)ml, D);
  misc::decide<<<1, misc::NT, 0, s>>>(st, c->dd.p, c->GWn.p, c->GW.p, (int)r, pl.prec == PREC_EXACT, c->recs.p, 1);
  CUK();
  c->launches += 2;
  tr.mark("e0");

  // one outer iteration = one graph; one conditional WHILE node per HALS side
  if (K > 0) {
    CU(cudaGraphCreate(&se->graph, 0));
    cudaGraphConditionalHandle ch = 0, cw = 0;
    const bool persist = hals_persistent(pl.prec, pl.r);
    if (pl.inner_h == ENMF_INNER_HALS && !persist)
      CU(cudaGraphConditionalHandleCreate(&ch, se->graph, 1, cudaGraphCondAssignDefault));
    if (pl.inner_w == ENMF_INNER_HALS && !persist)
      CU(cudaGraphConditionalHandleCreate(&cw, se->graph, 1, cudaGraphCondAssignDefault));
    const unsigned long long before = c->launches;
    CU(cudaStreamBeginCaptureToGraph(s, se->graph, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    try {
      enqueue_iteration(c, s, pl, ch, cw, INNER_CAPTURE, nullptr);
    } catch (...) {
      cudaGraph_t g2;
      cudaStreamEndCapture(s, &g2);
      close_session(c);
      throw;
    }
    cudaGraph_t g2;
    CU(cudaStreamEndCapture(s, &g2));
    const int hals_sides = (pl.inner_h == ENMF_INNER_HALS) + (pl.inner_w == ENMF_INNER_HALS);
    se->static_kernels = (int)(c->launches - before) - hals_sides * se->kps;
    c->launches = before;
    CU(cudaGraphInstantiate(&se->exec, se->graph, 0));
  }
  tr.mark("graph");
}

Session* need_session(enmf_gpu_ctx* c) {
  if (!c) throw Fail{ENMF_INVALID_ARGUMENT, "null context"};
  if (!c->sess) throw Fail{ENMF_INVALID_ARGUMENT, "no open run (call enmf_gpu_begin first)"};
  CU(cudaSetDevice(c->device));
  return c->sess;
}

size_t step_impl(enmf_gpu_ctx* c, uint64_t count) {
  Session* se = need_session(c);
  const size_t todo = (size_t)std::min<uint64_t>(count, se->K - se->launched);
  for (size_t k = 0; k < todo; ++k) CU(cudaGraphLaunch(se->exec, c->stream));
  se->launched += todo;
  return todo;
}

// One iteration with direct launches and CUDA events between phases.
void step_profiled_impl(enmf_gpu_ctx* c, double* phase_ms, size_t cap) {
  Session* se = need_session(c);
  if (se->launched >= se->K) throw Fail{ENMF_INVALID_ARGUMENT, "step_profiled: iteration budget exhausted"};
  Prof p{};
  for (auto& e : p.ev) CU(cudaEventCreate(&e));
  const unsigned long long before = c->launches;
  enqueue_iteration(c, c->stream, se->pl, 0, 0, INNER_HOSTLOOP, &p);
  c->launches = before;  // counted from the records at sync time
  CU(cudaStreamSynchronize(c->stream));
  se->launched += 1;
  double out[12] = {0};
  auto el = [&](int a, int b) {
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, p.ev[a], p.ev[b]));
    return (double)t;
  };
  out[0] = el(0, 1);   // iter_begin + gram(W_y) + reinit check
  out[1] = el(1, 2);   // W_yᵀ X
  out[2] = p.hals_ms[0] > 0 ? p.hals_ms[0] : el(2, 3);  // H update (sweeps only / BPP)
  out[3] = el(3, 4);   // H extrapolation
  out[4] = el(4, 5);   // gram(T) + reinit check
  out[5] = el(5, 6);   // T Xᵀ
  out[6] = p.hals_ms[1] > 0 ? p.hals_ms[1] : el(6, 7);  // W update
  out[7] = el(7, 8);   // error products
  out[8] = el(8, 9);   // decide + finalize
  out[9] = p.hals_sweeps[0];
  out[10] = p.hals_sweeps[1];
  for (auto& e : p.ev) cudaEventDestroy(e);
  for (size_t i = 0; i < cap && i < 11; ++i) phase_ms[i] = out[i];
}

size_t sync_impl(enmf_gpu_ctx* c, enmf_gpu_iter* iters, size_t cap, size_t* n_iters) {
  Session* se = need_session(c);
  DevState out;
  CU(cudaMemcpyAsync(&out, c->st.p, sizeof out, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  x_verdict(c, true);
  const size_t done = (size_t)out.k;
  std::vector<enmf_gpu_iter> recs(done + 1);
  CU(cudaMemcpy(recs.data(), c->recs.p, (done + 1) * sizeof(enmf_gpu_iter), cudaMemcpyDeviceToHost));
  // kernels actually executed: static part per iteration + the sweeps taken
  for (size_t k = se->counted + 1; k <= done; ++k) {
    unsigned long long sw = 0;
    if (se->pl.inner_h == ENMF_INNER_HALS) sw += recs[k].inner_h_count;
    if (se->pl.inner_w == ENMF_INNER_HALS) sw += recs[k].inner_w_count;
    c->launches += (unsigned long long)se->static_kernels + sw * se->kps;
  }
  se->counted = std::max(se->counted, done);
  const size_t count = done + 1;
  if (iters) std::memcpy(iters, recs.data(), std::min(count, cap) * sizeof(enmf_gpu_iter));
  if (n_iters) *n_iters = count;
  if (out.error_code != ENMF_OK) {
    se->failed = true;
    const char* what = out.error_code == ENMF_NON_FINITE ? "iteration produced a non-finite value"
                       : out.error_code == ENMF_NO_CONVERGENCE
                           ? "no convergence (degenerate factor column persists after reinitialization, or "
                             "active_set_solve exchange limit exceeded)"
                           : "device error";
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s at iteration %llu", what, (unsigned long long)out.k);
    throw Fail{out.error_code, buf};
  }
  return count;
}

void end_impl(enmf_gpu_ctx* c, double* w_out, double* h_out, double* norm_x_out) {
  Session* se = need_session(c);
  cudaStream_t s = c->stream;
  const size_t m = se->ml, n = se->nl, r = se->r;   // this rank's shards (the whole factors on one GPU)
  if (norm_x_out) {
    DevState out;
    CU(cudaMemcpyAsync(&out, c->st.p, sizeof out, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    *norm_x_out = out.norm_x;
  }
  if (w_out) {
    dim3 tb(32, 8), tg((unsigned)((m + 31) / 32), (unsigned)((r + 31) / 32));
    misc::transpose<<<tg, tb, 0, s>>>(c->WT.p, c->scratch.p, (int)r, (int)m);
    CUK();
    c->launches++;
    CU(cudaMemcpyAsync(w_out, c->scratch.p, m * r * 8,
                       se->dev_factors ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  }
  if (h_out)
    CU(cudaMemcpyAsync(h_out, c->H.p, r * n * 8, se->dev_factors ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       s));
  CU(cudaStreamSynchronize(s));
  close_session(c);
}

// enmf::run: begin + K steps + sync + end.
int solve_impl(enmf_gpu_ctx* c, const double* w0, const double* h0, size_t r, bool dev_factors,
               const enmf_gpu_config* cfg, enmf_gpu_iter* iters, size_t iters_cap, size_t* n_iters, double* w_out,
               double* h_out, double* norm_x_out) {
  begin_impl(c, w0, h0, r, dev_factors, cfg);
  try {
    step_impl(c, cfg->max_outer_iterations);
    sync_impl(c, iters, iters_cap, n_iters);
  } catch (...) {
    close_session(c);
    throw;
  }
  end_impl(c, w_out, h_out, norm_x_out);
  return ENMF_OK;
}

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const Fail& e) {
    set_err(e);
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ENMF_INVALID_ARGUMENT;
  }
}

}  // namespace

extern "C" {

int enmf_gpu_begin(enmf_gpu_ctx* c, const double* w0, const double* h0, size_t r, int factors_on_device,
                   const enmf_gpu_config* cfg) {
  return guard([&] {
    begin_impl(c, w0, h0, r, factors_on_device != 0, cfg);
    return ENMF_OK;
  });
}

int enmf_gpu_step(enmf_gpu_ctx* c, uint64_t count) {
  return guard([&] {
    step_impl(c, count);
    return ENMF_OK;
  });
}

int enmf_gpu_step_profiled(enmf_gpu_ctx* c, double* phase_ms, size_t cap) {
  return guard([&] {
    step_profiled_impl(c, phase_ms, cap);
    return ENMF_OK;
  });
}

int enmf_gpu_sync(enmf_gpu_ctx* c, enmf_gpu_iter* iters, size_t cap, size_t* n_iters) {
  return guard([&] {
    sync_impl(c, iters, cap, n_iters);
    return ENMF_OK;
  });
}

int enmf_gpu_end(enmf_gpu_ctx* c, double* w_out, double* h_out, double* norm_x) {
  return guard([&] {
    end_impl(c, w_out, h_out, norm_x);
    return ENMF_OK;
  });
}

void* enmf_gpu_stream(enmf_gpu_ctx* c) { return c ? (void*)c->stream : nullptr; }

int enmf_gpu_digit_levels(const enmf_gpu_ctx* c, int32_t* levels) {
  return guard([&] {
    if (!c || !levels) throw Fail{ENMF_INVALID_ARGUMENT, "digit_levels: bad arguments"};
    const bool d = c->dist != nullptr;
    const auto& wx = d ? c->xd_cols : c->xd_x;
    const auto& xt = d ? c->xd_rows : c->xd_xt;
    levels[0] = wx.ready ? wx.levels : 0;
    levels[1] = xt.ready ? xt.levels : 0;
    return ENMF_OK;
  });
}

}  // extern "C"

namespace enmf_host {
void set_last_error(const std::string& msg) { g_last_error = msg; }   // io.cpp's errors
}

#include "dist_api.inc"
#include "cabi.inc"
#include "kernels_api.inc"
#include "batch_api.inc"

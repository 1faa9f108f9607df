// gemm.cuh — FP64 contractions of the enmf hot path on sm_100a.
//
// One tensor-core kernel serves every dense contraction of step()
// (engine.hpp:309-440):
//   C_H  = W_yᵀ X       cross_wx   linalg.hpp:67-83    A = W_yᵀ (r×m), B = X   (K×N, N-contiguous)
//   P    = T Xᵀ = (X Tᵀ)ᵀ cross_xht linalg.hpp:107-124  A = T    (r×n), B = X   (N×K, K-contiguous)
//   G    = A Aᵀ         gram       linalg.hpp:49-64    A = W_yᵀ | T | W_nᵀ,  B = A (K-contiguous)
// Blackwell has no FP64 tcgen05 kind, so the FP64 tensor path is the legacy
// warp-level DMMA: PTX mma.sync.m8n8k4.f64, which ptxas lowers to one native
// DMMA.8x8x4 on sm_100a (measured 37.1 TFLOP/s peak on B200 vs 33.8 for DFMA,
// profiles/r01_fp64_peak.txt).  Tiles stream through a 3-stage cp.async ring
// in shared memory with bank-conflict-free padded layouts; split-K keeps all
// 148 SMs busy on the skinny r×32768 outputs and its partials are reduced in a
// fixed order (deterministic).
//
// The *_exact kernels are the bitwise-faithful debug path (precision =
// ENMF_PRECISION_FP64_EXACT): one thread per output element summing in the
// reference's sequential order with separately rounded multiply and add.
#pragma once

#include "common.cuh"
#include "tc.cuh"

namespace gemm {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3, NT = 256;
constexpr int LDA_S = BK + 4;   // A tile [m][k]
constexpr int LDB_N = BN + 4;   // B tile [k][n]   (B_KMAJOR = false)
constexpr int LDB_K = BK + 4;   // B tile [n][k]   (B_KMAJOR = true)
constexpr int A_STAGE = BM * LDA_S;
constexpr int B_STAGE = (BN * LDB_K > BK * LDB_N) ? BN * LDB_K : BK * LDB_N;
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * (int)sizeof(double);

ENMF_DEV void cp_async16(double* smem, const double* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
ENMF_DEV void cp_async8(double* smem, const double* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
ENMF_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
ENMF_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

ENMF_DEV void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct Params {
  const double* A; long lda;     // M×K, K contiguous
  const double* B; long ldb;     // B_KMAJOR: N×K (K contiguous) ; else K×N (N contiguous)
  double* C; long ldc;           // M×N
  int M, N, K;
  int splits;                    // split-K factor (gridDim.z)
  double* partials;              // splits × M × N (splits > 1)
  unsigned* counters;            // one per output tile (REDUCE_LAST)
  int sym;                       // write C[i][j] = C[j][i] from i <= j (Gram)
  const DevState* st;            // nullable: skip work when !st->active
};

// Loads one BM×BK tile of a K-contiguous operand (rows row0.., k0..).
template <int VEC>
ENMF_DEV void load_kmajor(double* s, int lds, const double* g, long ld, int rows_valid, int row0,
                          int k0, int K, int nrows) {
  constexpr int CH = BK / VEC;  // chunks per row
  for (int c = threadIdx.x; c < nrows * CH; c += blockDim.x) {
    const int row = c / CH, col = (c % CH) * VEC;
    const int gr = row0 + row, gk = k0 + col;
    int valid = 0;
    if (gr < rows_valid && gk < K) valid = (K - gk >= VEC) ? VEC : (K - gk);
    const double* src = valid ? g + (long)gr * ld + gk : g;
    if (VEC == 2) cp_async16(s + row * lds + col, src, valid * 8);
    else cp_async8(s + row * lds + col, src, valid * 8);
  }
}
// Loads a BK×BN tile of an N-contiguous operand (k rows k0.., cols n0..).
template <int VEC>
ENMF_DEV void load_nmajor(double* s, const double* g, long ld, int k0, int K, int n0, int N) {
  constexpr int CH = BN / VEC;
  for (int c = threadIdx.x; c < BK * CH; c += blockDim.x) {
    const int row = c / CH, col = (c % CH) * VEC;
    const int gk = k0 + row, gn = n0 + col;
    int valid = 0;
    if (gk < K && gn < N) valid = (N - gn >= VEC) ? VEC : (N - gn);
    const double* src = valid ? g + (long)gk * ld + gn : g;
    if (VEC == 2) cp_async16(s + row * LDB_N + col, src, valid * 8);
    else cp_async8(s + row * LDB_N + col, src, valid * 8);
  }
}

// C[M×N] (+)= A · op(B) on DMMA.  grid = (ceil(N/BN), ceil(M/BM), splits).
// WMW = warps along M (2: 8 warps of 64×32; 4: 16 warps of 32×32).
template <bool B_KMAJOR, int VEC, bool REDUCE_LAST, int WMW = 2>
__global__ void __launch_bounds__(WMW * 4 * 32, 1) gemm_f64_dmma(Params p) {
  constexpr int MI = 16 / WMW;          // 8-row m-tiles per warp
  constexpr int WROWS = BM / WMW;
  constexpr int NTH = WMW * 4 * 32;
  if (p.st && !dev_active(p.st)) return;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WMW, wn = warp / WMW;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int KB = (p.K + BK - 1) / BK;
  const int per = (KB + p.splits - 1) / p.splits;
  const int kb0 = blockIdx.z * per;
  const int kb1 = min(KB, kb0 + per);
  const int nk = max(0, kb1 - kb0);

  double acc[MI][4][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto issue = [&](int kb, int stage) {
    const int k0 = (kb0 + kb) * BK;
    load_kmajor<VEC>(As + stage * A_STAGE, LDA_S, p.A, p.lda, p.M, m0, k0, p.K, BM);
    if (B_KMAJOR) load_kmajor<VEC>(Bs + stage * B_STAGE, LDB_K, p.B, p.ldb, p.N, n0, k0, p.K, BN);
    else load_nmajor<VEC>(Bs + stage * B_STAGE, p.B, p.ldb, k0, p.K, n0, p.N);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kb + STAGES - 1;
      if (nxt < nk) issue(nxt, nxt % STAGES);
      cp_commit();
    }
    const double* as = As + (kb % STAGES) * A_STAGE + (wm * WROWS + g) * LDA_S + t;
    const double* bs = Bs + (kb % STAGES) * B_STAGE;
    // Fragments are double-buffered in registers (the loads for k-step kk+1 are
    // in flight while kk's DMMAs issue).
    double a[2][MI], b[2][4];
    auto load_frag = [&](int kk, int buf) {
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) a[buf][mi] = as[mi * 8 * LDA_S + kk * 4];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        if (B_KMAJOR) b[buf][ni] = bs[(wn * 32 + ni * 8 + g) * LDB_K + kk * 4 + t];
        else b[buf][ni] = bs[(kk * 4 + t) * LDB_N + wn * 32 + ni * 8 + g];
      }
    };
    load_frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int cur = kk & 1;
      if (kk + 1 < BK / 4) load_frag(kk + 1, cur ^ 1);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[cur][mi], b[cur][ni]);
    }
  }
  cp_wait<0>();

  // ---- epilogue ----
  const bool split = p.splits > 1;
  double* out = split ? p.partials + (long)blockIdx.z * p.M * p.N : p.C;
  const long ldo = split ? p.N : p.ldc;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int row = m0 + wm * WROWS + mi * 8 + g;
    if (row >= p.M) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int col = n0 + wn * 32 + ni * 8 + 2 * t;
      if (!split && p.sym) {
        // Gram without split: keep the upper triangle, mirror it.
        for (int e = 0; e < 2; ++e) {
          const int c = col + e;
          if (c < p.N && row <= c) {
            out[(long)row * ldo + c] = acc[mi][ni][e];
            out[(long)c * ldo + row] = acc[mi][ni][e];
          }
        }
      } else if (col + 1 < p.N && ((ldo & 1) == 0)) {
        *reinterpret_cast<double2*>(out + (long)row * ldo + col) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      } else {
        if (col < p.N) out[(long)row * ldo + col] = acc[mi][ni][0];
        if (col + 1 < p.N) out[(long)row * ldo + col + 1] = acc[mi][ni][1];
      }
    }
  }
  if (!split || !REDUCE_LAST) return;

  // Last CTA of this output tile sums the partials in split order 0..S-1.
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    unsigned* ctr = p.counters + blockIdx.y * gridDim.x + blockIdx.x;
    const unsigned prev = atomicAdd(ctr, 1u);
    s_last = (prev == (unsigned)p.splits - 1) ? 1u : 0u;
    if (s_last) *ctr = 0;  // re-arm for the next launch
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int rows = min(BM, p.M - m0), cols = min(BN, p.N - n0);
  const long MN = (long)p.M * p.N;
  for (int e = tid; e < rows * cols; e += NTH) {
    const int i = m0 + e / cols, j = n0 + e % cols;
    if (p.sym && i > j) continue;
    const double* src = p.partials + (long)i * p.N + j;
    double v = __ldcg(src);
    for (int s = 1; s < p.splits; ++s) v = __dadd_rn(v, __ldcg(src + s * MN));
    p.C[(long)i * p.ldc + j] = v;
    if (p.sym) p.C[(long)j * p.ldc + i] = v;
  }
}

// ---- small-tile variant: 64×64×16 CTA tile, 4 warps of 32×32, 3 stages --------
// 60 KB of shared memory and ≤ 128 registers, so THREE CTAs share an SM: a
// CTA waiting at its k-block barrier no longer drains the SM's DMMA pipe
// (the 128×128 single-CTA kernel above tops out at 79% DMMA-pipe activity,
// profiles/r01_gemm_ncu.txt).
// Tiles are stored unpadded with an XOR swizzle (16 KB per stage, 4 stages, still
// three CTAs per SM): K-major element (row, k) at row·BK + (k ^ 4·(row & 3)),
// N-major element (k, n) at k·BN + (n ^ nswz(k)); both keep 16-byte chunks whole
// and make the 8-byte fragment loads conflict-free.
namespace st {
constexpr int BM = 64, BN = 64, BK = 16, STAGES = 4, NTH = 128;
constexpr int LDA_S = BK;
constexpr int LDB_N = BN;
constexpr int LDB_K = BK;
constexpr int A_STAGE = BM * LDA_S;
constexpr int B_STAGE = (BN * LDB_K > BK * LDB_N) ? BN * LDB_K : BK * LDB_N;
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * (int)sizeof(double);
ENMF_DEV int kswz(int row) { return 4 * (row & 3); }
ENMF_DEV int nswz(int k) { return 4 * (k & 1) + 8 * ((k >> 1) & 1); }
}  // namespace st

template <int VEC, int BKk, int NTHk>
ENMF_DEV void st_load_kmajor(double* s, int lds, const double* g, long ld, int rows_valid, int row0, int k0,
                             int K, int nrows) {
  constexpr int CH = BKk / VEC;
  for (int c = threadIdx.x; c < nrows * CH; c += NTHk) {
    const int row = c / CH, col = (c % CH) * VEC;
    const int gr = row0 + row, gk = k0 + col;
    int valid = 0;
    if (gr < rows_valid && gk < K) valid = (K - gk >= VEC) ? VEC : (K - gk);
    const double* src = valid ? g + (long)gr * ld + gk : g;
    double* d = s + row * lds + (col ^ st::kswz(row));
    if (VEC == 2) cp_async16(d, src, valid * 8);
    else cp_async8(d, src, valid * 8);
  }
}
template <int VEC>
ENMF_DEV void st_load_nmajor(double* s, const double* g, long ld, int k0, int K, int n0, int N) {
  constexpr int CH = st::BN / VEC;
  for (int c = threadIdx.x; c < st::BK * CH; c += st::NTH) {
    const int row = c / CH, col = (c % CH) * VEC;
    const int gk = k0 + row, gn = n0 + col;
    int valid = 0;
    if (gk < K && gn < N) valid = (N - gn >= VEC) ? VEC : (N - gn);
    const double* src = valid ? g + (long)gk * ld + gn : g;
    double* d = s + row * st::LDB_N + (col ^ st::nswz(row));
    if (VEC == 2) cp_async16(d, src, valid * 8);
    else cp_async8(d, src, valid * 8);
  }
}

// Epilogue of the 64×64 DMMA kernels: the warp's 32×32 accumulators to C (or to this split's
// partial slice), and with REDUCE_LAST the last split CTA of a tile sums the slices in order.
template <bool REDUCE_LAST>
ENMF_DEV void st_epilogue(const Params& p, const double (&acc)[4][4][2], int m0, int n0, int wm, int wn, int g, int t) {
  constexpr int BM = st::BM, BN = st::BN, NTH = st::NTH;
  const int tid = threadIdx.x;
  const bool split = p.splits > 1;
  double* out = split ? p.partials + (long)blockIdx.z * p.M * p.N : p.C;
  const long ldo = split ? p.N : p.ldc;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int row = m0 + wm * 32 + mi * 8 + g;
    if (row >= p.M) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int col = n0 + wn * 32 + ni * 8 + 2 * t;
      if (!split && p.sym) {
        for (int e = 0; e < 2; ++e) {
          const int c = col + e;
          if (c < p.N && row <= c) {
            out[(long)row * ldo + c] = acc[mi][ni][e];
            out[(long)c * ldo + row] = acc[mi][ni][e];
          }
        }
      } else if (col + 1 < p.N && ((ldo & 1) == 0)) {
        *reinterpret_cast<double2*>(out + (long)row * ldo + col) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      } else {
        if (col < p.N) out[(long)row * ldo + col] = acc[mi][ni][0];
        if (col + 1 < p.N) out[(long)row * ldo + col + 1] = acc[mi][ni][1];
      }
    }
  }
  if (!split || !REDUCE_LAST) return;
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    unsigned* ctr = p.counters + blockIdx.y * gridDim.x + blockIdx.x;
    const unsigned prev = atomicAdd(ctr, 1u);
    s_last = (prev == (unsigned)p.splits - 1) ? 1u : 0u;
    if (s_last) *ctr = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int rows = min(BM, p.M - m0), cols = min(BN, p.N - n0);
  const long MN = (long)p.M * p.N;
  for (int e = tid; e < rows * cols; e += NTH) {
    const int i = m0 + e / cols, j = n0 + e % cols;
    if (p.sym && i > j) continue;
    const double* src = p.partials + (long)i * p.N + j;
    double v = __ldcg(src);
    for (int s = 1; s < p.splits; ++s) v = __dadd_rn(v, __ldcg(src + s * MN));
    p.C[(long)i * p.ldc + j] = v;
    if (p.sym) p.C[(long)j * p.ldc + i] = v;
  }
}

template <bool B_KMAJOR, int VEC, bool REDUCE_LAST>
__global__ void __launch_bounds__(st::NTH, 3) gemm_f64_dmma_s(Params p) {
  constexpr int BM = st::BM, BN = st::BN, BK = st::BK, STAGES = st::STAGES, NTH = st::NTH;
  constexpr int LDA_S = st::LDA_S, LDB_N = st::LDB_N, LDB_K = st::LDB_K;
  constexpr int A_STAGE = st::A_STAGE, B_STAGE = st::B_STAGE;
  if (p.st && !dev_active(p.st)) return;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;     // 2×2 warps of 32×32
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;   // grid = (M tiles, N tiles, splits)
  const int KB = (p.K + BK - 1) / BK;
  const int per = (KB + p.splits - 1) / p.splits;
  const int kb0 = blockIdx.z * per;
  const int kb1 = min(KB, kb0 + per);
  const int nk = max(0, kb1 - kb0);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Interior tiles (the whole tile in range, K a multiple of BK, 16-byte rows): every
  // thread's four 16-byte chunks per operand have fixed addresses up to the k offset.
  const bool full = VEC == 2 && m0 + BM <= p.M && n0 + BN <= p.N && (p.K % BK) == 0;
  const double* fa = p.A + (long)(m0 + (tid >> 3)) * p.lda + (long)kb0 * BK + (tid & 7) * 2;
  const int sa = (tid >> 3) * LDA_S + (((tid & 7) * 2) ^ st::kswz(tid >> 3));
  const double* fb = B_KMAJOR ? p.B + (long)(n0 + (tid >> 3)) * p.ldb + (long)kb0 * BK + (tid & 7) * 2
                              : p.B + (long)(kb0 * BK + (tid >> 5)) * p.ldb + n0 + (tid & 31) * 2;
  const int sb = B_KMAJOR ? (tid >> 3) * LDB_K + (((tid & 7) * 2) ^ st::kswz(tid >> 3))
                          : (tid >> 5) * LDB_N + (((tid & 31) * 2) ^ st::nswz(tid >> 5));
  auto issue = [&](int kb, int stage) {
    if (full) {
      double* da = As + stage * A_STAGE + sa;
      double* db = Bs + stage * B_STAGE + sb;
      const double* ga = fa + (long)kb * BK;
#pragma unroll
      for (int i = 0; i < 4; ++i) cp_async16(da + i * 16 * LDA_S, ga + (long)i * 16 * p.lda, 16);
      if (B_KMAJOR) {
        const double* gb = fb + (long)kb * BK;
#pragma unroll
        for (int i = 0; i < 4; ++i) cp_async16(db + i * 16 * LDB_K, gb + (long)i * 16 * p.ldb, 16);
      } else {
        const double* gb = fb + (long)kb * BK * p.ldb;
#pragma unroll
        for (int i = 0; i < 4; ++i) cp_async16(db + i * 4 * LDB_N, gb + (long)i * 4 * p.ldb, 16);
      }
      return;
    }
    const int k0 = (kb0 + kb) * BK;
    st_load_kmajor<VEC, BK, NTH>(As + stage * A_STAGE, LDA_S, p.A, p.lda, p.M, m0, k0, p.K, BM);
    if (B_KMAJOR) st_load_kmajor<VEC, BK, NTH>(Bs + stage * B_STAGE, LDB_K, p.B, p.ldb, p.N, n0, k0, p.K, BN);
    else st_load_nmajor<VEC>(Bs + stage * B_STAGE, p.B, p.ldb, k0, p.K, n0, p.N);
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kb + STAGES - 1;
      if (nxt < nk) issue(nxt, nxt % STAGES);
      cp_commit();
    }
    // rows wm·32 + mi·8 + g (K-major) share row & 3 = g & 3; N-major k-rows kk·4 + t share k & 3 = t
    const double* as = As + (kb % STAGES) * A_STAGE + (wm * 32 + g) * LDA_S;
    const double* bs = Bs + (kb % STAGES) * B_STAGE;
    double a[2][4], b[2][4];
    auto load_frag = [&](int kk, int buf) {
      const int kq = 4 * (kk ^ (g & 3)) + t;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[buf][mi] = as[mi * 8 * LDA_S + kq];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        if (B_KMAJOR) b[buf][ni] = bs[(wn * 32 + ni * 8 + g) * LDB_K + kq];
        else b[buf][ni] = bs[(kk * 4 + t) * LDB_N + ((wn * 32 + ni * 8 + g) ^ st::nswz(t))];
      }
    };
    load_frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int cur = kk & 1;
      if (kk + 1 < BK / 4) load_frag(kk + 1, cur ^ 1);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[cur][mi], b[cur][ni]);
    }
  }
  cp_wait<0>();

  st_epilogue<REDUCE_LAST>(p, acc, m0, n0, wm, wn, g, t);
}

// Separate split-K reduction (fixed order), used when one output tile has
// many splits (the r×r Grams: K = 32768, 1 tile, 148 splits).
__global__ void reduce_splits(const double* __restrict__ part, int splits, int M, int N,
                              double* __restrict__ C, long ldc, int sym, const DevState* st) {
  if (st && !dev_active(st)) return;
  const long MN = (long)M * N;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < MN; e += (long)gridDim.x * blockDim.x) {
    const int i = (int)(e / N), j = (int)(e % N);
    if (sym && i > j) continue;
    double v = part[e];
    for (int s = 1; s < splits; ++s) v = __dadd_rn(v, part[e + s * MN]);
    C[(long)i * ldc + j] = v;
    if (sym) C[(long)j * ldc + i] = v;
  }
}

// ---- bitwise-faithful kernels (reference summation order, no FMA) --------

// gram (linalg.hpp:49-64) of the K×r matrix whose column k is row k of A
// (A r×K, K contiguous):  g[k][j] = sum_i A[k][i]*A[j][i], i ascending, k<=j, mirrored.
__global__ void gram_exact(const double* __restrict__ A, long lda, int r, int K, double* __restrict__ G,
                           const DevState* st) {
  if (st && !dev_active(st)) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= r * r) return;
  const int k = idx / r, j = idx % r;
  if (k > j) return;
  const double* ak = A + (long)k * lda;
  const double* aj = A + (long)j * lda;
  double s = 0.0;
  for (int i = 0; i < K; ++i) s = __dadd_rn(s, __dmul_rn(ak[i], aj[i]));
  G[k * r + j] = s;
  G[j * r + k] = s;
}

// cross_wx (linalg.hpp:67-83): out[k][j] = sum_i W[i][k]*X[i][j], i ascending; W given as WT (r×m).
__global__ void cross_wx_exact(const double* __restrict__ WT, const double* __restrict__ X, int m, int n,
                               int r, double* __restrict__ out, const DevState* st) {
  if (st && !dev_active(st)) return;
  const long idx = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (idx >= (long)r * n) return;
  const int k = (int)(idx / n), j = (int)(idx % n);
  const double* wk = WT + (long)k * m;
  double s = 0.0;
  for (int i = 0; i < m; ++i) s = __dadd_rn(s, __dmul_rn(wk[i], X[(long)i * n + j]));
  out[idx] = s;
}

// cross_xht (linalg.hpp:107-124): xht[i][k] = sum_j X[i][j]*T[k][j], j ascending;
// written transposed: P[k][i].
__global__ void cross_xht_exact(const double* __restrict__ X, const double* __restrict__ T, int m, int n,
                                int r, double* __restrict__ P, const DevState* st) {
  if (st && !dev_active(st)) return;
  const long idx = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (idx >= (long)r * m) return;
  const int k = (int)(idx / m), i = (int)(idx % m);
  const double* xi = X + (long)i * n;
  const double* tk = T + (long)k * n;
  double s = 0.0;
  for (int j = 0; j < n; ++j) s = __dadd_rn(s, __dmul_rn(xi[j], tk[j]));
  P[idx] = s;
}

// ---- the same kernel fed by TMA -----------------------------------------------------------
// Operand tiles arrive by cp.async.bulk.tensor (one elected thread, mbarrier completion) in the
// hardware's SWIZZLE_128B layout: a K-major tile is 64 rows × 16 doubles (one 128-byte row per
// tile row, its 16-byte chunks XOR-permuted by row % 8), an N-major B tile four 16 × 16 boxes.
// The 8-byte fragment loads follow the same permutation, so they stay conflict-free (K-major:
// the 8 rows of a fragment touch 8 distinct chunk positions).  Out-of-range elements are filled
// with zeros by the TMA unit — partial tiles need no separate load path.  Four stages, the
// slots released by each warp's arrive on an "empty" mbarrier; split-K and the epilogue as in
// gemm_f64_dmma_s.
namespace tm {
constexpr int A_BYTES = st::BM * st::BK * 8, B_BYTES = st::BN * st::BK * 8;
constexpr int SMEM_BYTES = 1024 + st::STAGES * (A_BYTES + B_BYTES) + 2 * st::STAGES * 8;
// element (row, k) of a K-major tile: row·16 + ((k/2) ^ (row % 8))·2 + k % 2
ENMF_DEV int kidx(int row, int k) { return row * 16 + ((((k >> 1) ^ (row & 7)) << 1) | (k & 1)); }
}  // namespace tm

template <bool B_KMAJOR, bool REDUCE_LAST>
__global__ void __launch_bounds__(st::NTH, 3) gemm_f64_dmma_t(Params p, const __grid_constant__ CUtensorMap ta,
                                                                const __grid_constant__ CUtensorMap tb) {
  constexpr int BM = st::BM, BN = st::BN, BK = st::BK, STAGES = st::STAGES;
  if (p.st && !dev_active(p.st)) return;
  extern __shared__ uint8_t smem_raw_t[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw_t) + 1023) & ~uintptr_t(1023));
  double* As = reinterpret_cast<double*>(sm);
  double* Bs = reinterpret_cast<double*>(sm + STAGES * tm::A_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * (tm::A_BYTES + tm::B_BYTES));
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 1, wn = warp >> 1;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int KB = (p.K + BK - 1) / BK;
  const int per = (KB + p.splits - 1) / p.splits;
  const int kb0 = blockIdx.z * per;
  const int nk = max(0, min(KB, kb0 + per) - kb0);
  if (tid == 0) {
    tc::prefetch_tmap(&ta);
    tc::prefetch_tmap(&tb);
    for (int s2 = 0; s2 < STAGES; ++s2) {
      tc::mbar_init(full + s2, 1);
      tc::mbar_init(empty + s2, st::NTH / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int kb, int s2) {
    const int k0 = (kb0 + kb) * BK;
    tc::mbar_expect_tx(full + s2, (uint32_t)(tm::A_BYTES + tm::B_BYTES));
    tc::tma_load_2d(As + s2 * BM * BK, &ta, full + s2, k0, m0);
    if (B_KMAJOR) {
      tc::tma_load_2d(Bs + s2 * BN * BK, &tb, full + s2, k0, n0);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) tc::tma_load_2d(Bs + s2 * BN * BK + q * 256, &tb, full + s2, n0 + 16 * q, k0);
    }
  };
  if (tid == 0)
    for (int s2 = 0; s2 < STAGES - 1 && s2 < nk; ++s2) issue(s2, s2);

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kb = 0; kb < nk; ++kb) {
    const int s2 = kb % STAGES;
    if (tid == 0 && kb + STAGES - 1 < nk) {     // refill the slot consumed at kb - 1
      const int sn = (kb + STAGES - 1) % STAGES;
      if (kb >= 1) tc::mbar_wait(empty + sn, (uint32_t)(((kb - 1) / STAGES) & 1));
      issue(kb + STAGES - 1, sn);
    }
    tc::mbar_wait(full + s2, (uint32_t)((kb / STAGES) & 1));
    const double* as = As + s2 * BM * BK;
    const double* bs = Bs + s2 * BN * BK;
    double a[2][4], b[2][4];
    auto load_frag = [&](int kk, int buf) {
      const int k = 4 * kk + t;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[buf][mi] = as[tm::kidx(wm * 32 + mi * 8 + g, k)];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        if (B_KMAJOR) {
          b[buf][ni] = bs[tm::kidx(wn * 32 + ni * 8 + g, k)];
        } else {               // box q = n / 16, row k, column c = n % 16 (16 doubles per row)
          const int c = (ni & 1) * 8 + g;
          b[buf][ni] = bs[(wn * 2 + (ni >> 1)) * 256 + k * 16 + ((((c >> 1) ^ (k & 7)) << 1) | (c & 1))];
        }
      }
    };
    load_frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int cur = kk & 1;
      if (kk + 1 < BK / 4) load_frag(kk + 1, cur ^ 1);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[cur][mi], b[cur][ni]);
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(empty + s2);  // this warp is done with the slot
  }
  st_epilogue<REDUCE_LAST>(p, acc, m0, n0, wm, wn, g, t);
}

}  // namespace gemm

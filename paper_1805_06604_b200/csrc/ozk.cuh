// ozk.cuh — the INT8-digit cross products on hand-written tcgen05 kernels.
//
// W_yᵀX and T·Xᵀ (linalg.hpp:67-83, 107-124) in FP64 accuracy from 8-bit digits
// (the splitting scheme of ozaki.cuh: every operand row scaled by a power of two into
// (-1/2, 1/2), D_0 ∈ [-128, 127] and offset digits d_p = D_p − 128, p ≥ 1), with all
// S(S+1)/2 digit pairs of an X tile formed in ONE kernel:
//
//   * both operands K-major in a chunked digit layout [K/32][SMAX][rows][32 bytes]:
//     one 4-D TMA box (32 B × rows × S digits × 1 chunk) lands a stage's S digit
//     tiles of an operand in shared memory as S SWIZZLE_32B K-major tiles, and reads
//     contiguous runs of rows·32 bytes per digit from HBM;
//   * M = 128 factor rows (r ≤ 128 per M block), N = BN = 64 X rows per tile, K = 32
//     per tcgen05.mma.kind::i8; the pairs (p, q) are summed per LEVEL ℓ = p + q in
//     TMEM (S accumulators of 128 lanes × BN int32 columns: 384 of 512 columns at S = 6),
//     so the digit products never leave the SM;
//   * K is cut into units of ≤ 8192 (256 chunks): a level sum over one unit is exact
//     in int32 (|d_p·d_q| ≤ 2^14, ≤ 7 pairs per level: < 2^30); the epilogue reads the
//     S level sums (tcgen05.ld), forms Σ_ℓ 2^{-8ℓ} L_ℓ in FP64 and writes one FP64
//     partial per unit;
//   * `finish` adds the unit partials in fixed order, the exact offset corrections
//     (c_q·rowsum(d^A_p) + c_p·colsum(d^B_q) + c_p·c_q·K, from the digit sums along the
//     contracted index) and the truncation-bias estimate of ozaki::combine, and scales
//     by the two exponents.
//
// Warp roles (persistent, one CTA per SM, units kq-major so the CTAs in flight read
// the same factor chunk from L2): warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA
// issuer, warps 2-5 = epilogue (TMEM lane quarter = warp % 4).
#pragma once

#include <cstdint>

#include "common.cuh"
#include "ozaki.cuh"
#include "tc.cuh"

namespace ozk {

constexpr int SMAX = ozaki::SMAX;   // digits cut per operand
constexpr int KC = 32;              // bytes (= int8 elements) of K per chunk / per MMA
constexpr int UNIT_CHUNKS = 512;    // K per unit ≤ 16384: level sums exact in int32 (≤ 7 pairs · 2^14 · 2^14 < 2^31)
constexpr int EPI_THREADS = 128;
constexpr int THREADS = 64 + EPI_THREADS;
constexpr int SMEM_LIMIT = 232448;  // sm_100 opt-in dynamic shared memory per block
constexpr int PF = 12;              // stages of L2 prefetch ahead of the shared-memory pipeline

// Digit operand layout = the shared-memory image of the MMA operand tiles: for K chunk c (32 of
// K) and row tile t (128 rows), the SMAX digit tiles are contiguous (SMAX × 4 KB), each the
// canonical no-swizzle K-major layout of 128 rows × 32 B: core matrices of 8 rows × 16 B
// ordered [row group (16)][K half (2)] — so one stage of an operand is ONE contiguous bulk copy.
constexpr int TROWS = 128;                  // rows per tile (M of the factor, N of the X tile)
constexpr int TILE = TROWS * KC;            // 4 KB
ENMF_DEV long tile_base(long ntiles, long row, long c, int q) { return ((c * ntiles + row / TROWS) * SMAX + q) * (long)TILE; }
ENMF_DEV int tile_off(int r, int kh) { return ((r >> 3) * 2 + kh) * 128 + (r & 7) * 16; }   // row r % 128, K half

// ---- digit cuts into the chunked layout ------------------------------------------
// 32 consecutive values v[0..31] (one chunk of one operand row) scaled by 2^-(e+1): the
// SMAX digit rows of 32 bytes each into their tiles (two 16-byte core-matrix rows); adds the digits
// into acc (valid elements only; the padding past K is stored as zero digits, which add
// nothing to any digit product and are not counted in the sums).
ENMF_DEV void cut_chunk(const double (&v)[32], int nvalid, double scale, int8_t* out, long rows, long row, long c,
                        int (&acc)[SMAX]) {
  uint32_t w[SMAX][8];
#pragma unroll
  for (int q = 0; q < SMAX; ++q)
#pragma unroll
    for (int t = 0; t < 8; ++t) w[q][t] = 0;
#pragma unroll
  for (int u = 0; u < 32; ++u) {
    int8_t dd[SMAX];
    int dig[SMAX];
    ozaki::cut8(v[u] * scale, dd, 1, dig);
    const bool ok = u < nvalid;
#pragma unroll
    for (int q = 0; q < SMAX; ++q) {
      acc[q] += ok ? dig[q] : 0;
      w[q][u >> 2] |= (ok ? (uint32_t)(uint8_t)dd[q] : 0u) << (8 * (u & 3));
    }
  }
  const long nt = (rows + TROWS - 1) / TROWS;
  const int r = (int)(row % TROWS);
#pragma unroll
  for (int q = 0; q < SMAX; ++q) {
    int8_t* t = out + tile_base(nt, row, c, q);
    *reinterpret_cast<uint4*>(t + tile_off(r, 0)) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
    *reinterpret_cast<uint4*>(t + tile_off(r, 1)) = make_uint4(w[q][4], w[q][5], w[q][6], w[q][7]);
  }
}

ENMF_DEV double pow2_neg(int e1) { return __longlong_as_double((long long)(1023 - e1) << 52); }   // 2^-e1

// Row-scaled operand: `rows` rows of a (row-major, lda), exponent per row from e_row (or, when
// amax != nullptr, from the row's |max| bit pattern — the per-product factor path, which also
// publishes the exponent into e_row).  Thread = (row, chunk group); grid.x over row blocks of
// blockDim.x, grid.y over chunk groups.  sums[q·rows + row] (zeroed by the caller) += digit sums.
__global__ void split_rows_chunked(const double* __restrict__ a, long rows, long K, long lda, int* e_row,
                                   const unsigned long long* amax, int8_t* __restrict__ out, int* __restrict__ sums,
                                   const DevState* st) {
  if (st && !dev_active(st)) return;
  const long row = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  int e;
  if (amax) {
    e = ozaki::exp_above(__longlong_as_double((long long)amax[row]));
    if (blockIdx.y == 0) e_row[row] = e;
  } else {
    e = e_row[row];
  }
  const double scale = pow2_neg(e + 1);
  const long nkc = (K + KC - 1) / KC;
  const double* ar = a + row * lda;
  const bool vec = ((reinterpret_cast<uintptr_t>(ar) & 15) == 0);
  int acc[SMAX] = {};
  for (long c = blockIdx.y; c < nkc; c += gridDim.y) {
    const long k0 = c * KC;
    const int nvalid = (int)min((long)KC, K - k0);
    double v[32];
    if (vec && nvalid == KC) {
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(ar + k0) + h);
        v[2 * h] = t.x;
        v[2 * h + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = u < nvalid ? ar[k0 + u] : 0.0;
    }
    cut_chunk(v, nvalid, scale, out, rows, row, c, acc);
  }
#pragma unroll
  for (int q = 0; q < SMAX; ++q) atomicAdd(sums + (long)q * rows + row, acc[q]);
}

// Column-scaled operand: the rows of the digit matrix are the COLUMNS j of x (R × C,
// row-major, ld), contracted over x's rows; exponent per column e_col[j].  Thread = (column,
// chunk group): each chunk reads 32 rows of one column (coalesced across the warp) and
// writes 32 contiguous bytes per digit.  sums[q·C + j] += digit sums.
__global__ void split_cols_chunked(const double* __restrict__ x, long R, long C, long ld, const int* __restrict__ e_col,
                                   int8_t* __restrict__ out, int* __restrict__ sums) {
  const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= C) return;
  const double scale = pow2_neg(e_col[j] + 1);
  const long nkc = (R + KC - 1) / KC;
  int acc[SMAX] = {};
  for (long c = blockIdx.y; c < nkc; c += gridDim.y) {
    const long i0 = c * KC;
    const int nvalid = (int)min((long)KC, R - i0);
    double v[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = u < nvalid ? __ldcs(x + (i0 + u) * ld + j) : 0.0;
    cut_chunk(v, nvalid, scale, out, C, j, c, acc);
  }
#pragma unroll
  for (int q = 0; q < SMAX; ++q) atomicAdd(sums + (long)q * C + j, acc[q]);
}

// ---- the digit GEMM ---------------------------------------------------------------
struct GemmArgs {
  const int8_t* A;   // factor digits (tile layout, nta row tiles)
  const int8_t* B;   // X digits (tile layout, ntb row tiles)
  int nta, ntb;
  int R, N;          // factor rows, X rows of the digit operands
  int nkc;           // 32-chunks of K (padded)
  int unit_chunks;   // chunks per unit (≤ UNIT_CHUNKS)
  int nkq, nmb, ntn; // units along K, M blocks of 128, N tiles of BN
  double* ws;        // CL × nkq × R × N FP64 partials (one slice per level group)
  const DevState* st;
};

ENMF_DEV double p2m(int e) { return __longlong_as_double((long long)(1023 - e) << 52); }   // 2^-e, 0 <= e < 1023

// One tcgen05.mma.cta_group::2.kind::i8 (M = 256, N = 128, K = 32) multiplies ONE X digit tile q
// (B: the tile's 128 X rows split 64 / 64 over the two CTAs' shared memory, read by both tensor
// cores) by TWO different factor digits at once: the A operand at the same shared-memory offset
// holds digit p in CTA 0 and digit p + 1 in CTA 1, so CTA 0 accumulates pair (p, q) into its
// level-(p+q) slot while CTA 1 accumulates (p+1, q) into its level-(p+q+1) slot.  TMEM slot j
// holds level 2j in CTA 0 and 2j+1 in CTA 1 (J = ⌈S/2⌉ slots of 128 columns).  Per K chunk the
// S(S+1)/2 pairs take 12 pair-MMAs at S = 6 (19 at S = 7; the few half-empty ones multiply a
// zero A tile).
//
// Why (replacing a level-split kernel that multicast every digit tile of a stage to both CTAs of
// a pair, each CTA forming 10-11 of the 21 pairs with cta_group::1 MMAs): each X digit tile now
// reaches shared memory once, as its two halves, so a stage is 2 × (S factor tiles + S half X
// tiles) = 72 KB per 128 X rows × 32 of K instead of 96 KB, and the tensor cores read 6 KB of
// shared memory per 64-cycle MMA instead of 8 KB.  Measured at C5: 2.07 → 1.92 ms per product
// (ncu), tensor pipe 61 → 87% active (profiles/r02_ozk_gemm_ncu.txt, r02_ozk_pair_ncu.txt); the
// pair layout was checked against the host first (tools/probe/umma2_probe.cu).
//
// Roles (per CTA, 192 threads): warp 0 = TMA producer (both CTAs: the S factor tiles into slots
// shifted by one in CTA 1, and this CTA's S half X tiles); warp 1 = MMA issuer in CTA 0, and in
// CTA 1 the forwarder that tells CTA 0's issuer its half of the stage has landed; warps 2-5 =
// epilogue (each CTA reads its own slots).  The MMA commits free the stage / publish the
// accumulators in both CTAs (multicast); both CTAs' epilogues release the accumulators to CTA 0.
template <int S>
struct PairCfg {
  static constexpr int J = (S + 1) / 2;                // accumulator slots (levels 2j + rank)
  static constexpr int A_SLOTS = S + 1;                // digit tiles −1..S−1 (rank 0) / 0..S (rank 1)
  static constexpr int A_BYTES = A_SLOTS * TILE;
  static constexpr int B_HALF = TILE / 2;              // 64 X rows × 32 B (the first / second half of a tile)
  static constexpr int B_BYTES = S * B_HALF;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int NS = (SMEM_LIMIT - 4096) / STAGE > 8 ? 8 : (SMEM_LIMIT - 4096) / STAGE;
  static constexpr int SMEM = 1024 + NS * STAGE + 1024;
  static constexpr int TMEM_COLS = 512;
  static_assert(J * TROWS <= 512, "level slots must fit the TMEM columns");
  static_assert(NS >= 3, "pipeline too shallow");
};

ENMF_DEV uint32_t peer0(const void* p) {               // CTA 0's shared::cluster address of p
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(tc::smem_u32(p)));
  return r;
}
// relaxed: what it announces (bulk copies landed / TMEM loads waited) is already ordered by the
// mbarrier wait / tcgen05.wait it follows; a release here costs a full GPU membar per stage
ENMF_DEV void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
ENMF_DEV void mma_i8_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
ENMF_DEV void commit_pair(uint64_t* b) {               // arrive on b in both CTAs of the pair
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                   tc::smem_u32(b)),
               "h"((uint16_t)3)
               : "memory");
}

template <int S>
__global__ void __launch_bounds__(THREADS, 1) gemm_pair(GemmArgs g) {
  using C = PairCfg<S>;
  if (g.st && !dev_active(g.st)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                  // NS × A_BYTES
  uint8_t* sB = smem + C::NS * C::A_BYTES;             // NS × B_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::NS * C::STAGE);
  uint64_t* full = bars;                               // this CTA's half of the stage landed
  uint64_t* pfull = bars + C::NS;                      // (CTA 0) CTA 1's half landed
  uint64_t* empty = bars + 2 * C::NS;                  // the pair-MMAs are done with the stage
  uint64_t* tfull = bars + 3 * C::NS;                  // accumulators complete
  uint64_t* tempty = tfull + 1;                        // (CTA 0) both epilogues drained them
  uint32_t* tbase_s = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)tc::cluster_rank();
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  // the A slot no digit lands in stays zero: slot 0 (digit −1) in CTA 0, slot S (digit S) in CTA 1
  {
    const int zs = rank == 0 ? 0 : S;
    for (int st = 0; st < C::NS; ++st)
      for (int e = threadIdx.x; e < TILE / 16; e += THREADS)
        reinterpret_cast<uint4*>(sA + st * C::A_BYTES + zs * TILE)[e] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NS; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(pfull + s, 1);
      tc::mbar_init(empty + s, 1);
    }
    tc::mbar_init(tfull, 1);
    tc::mbar_init(tempty, 2 * (EPI_THREADS / 32));
    tc::fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc::smem_u32(tbase_s)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc::fence_before();
  tc::cluster_sync();                                  // barriers, zero tiles and TMEM ready in both CTAs
  tc::fence_after();
  const uint32_t tbase = *tbase_s;

  const int items = g.nkq * g.nmb * g.ntn;
  if (warp == 0) {                                     // ---- TMA producer (both CTAs)
    int stage = 0;
    uint32_t phase = 0;
    for (int w = cluster; w < items; w += nclusters) {
      const int kq = w / (g.nmb * g.ntn), rem = w % (g.nmb * g.ntn);
      const int mb = rem / g.ntn, tn = rem % g.ntn;
      const int c0 = kq * g.unit_chunks, c1 = min(g.nkc, c0 + g.unit_chunks);
      for (int c = c0; c < c1; ++c) {
        tc::mbar_wait(empty + stage, phase ^ 1);
        if (tc::elect_one()) {
          tc::mbar_expect_tx(full + stage, (uint32_t)(S * TILE + S * C::B_HALF));
          const int8_t* asrc = g.A + ((long)c * g.nta + mb) * SMAX * TILE;
          const int8_t* bsrc = g.B + ((long)c * g.ntb + tn) * SMAX * TILE + rank * C::B_HALF;
          tc::bulk_load(sA + stage * C::A_BYTES + (rank == 0 ? TILE : 0), asrc, (uint32_t)(S * TILE), full + stage);
#pragma unroll
          for (int q = 0; q < S; ++q)
            tc::bulk_load(sB + stage * C::B_BYTES + q * C::B_HALF, bsrc + (long)q * TILE, (uint32_t)C::B_HALF,
                          full + stage);
          // the X digits stream from HBM exactly once: pull them PF stages ahead into L2
          if (rank == 0 && c + PF < c1)
            tc::bulk_prefetch_l2(g.B + ((long)(c + PF) * g.ntb + tn) * SMAX * TILE, (uint32_t)(S * TILE));
        }
        __syncwarp();
        if (++stage == C::NS) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && rank == 1) {                 // ---- CTA 1: forward "my half landed" to CTA 0
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t pf0 = peer0(pfull);
    for (int w = cluster; w < items; w += nclusters) {
      const int kq = w / (g.nmb * g.ntn);
      const int c0 = kq * g.unit_chunks, c1 = min(g.nkc, c0 + g.unit_chunks);
      for (int c = c0; c < c1; ++c) {
        tc::mbar_wait(full + stage, phase);
        if (tc::elect_one()) arrive_remote(pf0 + stage * 8);
        __syncwarp();
        if (++stage == C::NS) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {                              // ---- CTA 0: the pair-MMA issuer
    constexpr uint32_t IDESC = tc::idesc_i8(256, TROWS);
    const uint64_t dA0 = tc::desc_noswz(tc::smem_u32(sA), 128, 256);
    const uint64_t dB0 = tc::desc_noswz(tc::smem_u32(sB), 128, 256);
    int stage = 0;
    uint32_t phase = 0, tph = 0;
    for (int w = cluster; w < items; w += nclusters) {
      const int kq = w / (g.nmb * g.ntn);
      const int c0 = kq * g.unit_chunks, c1 = min(g.nkc, c0 + g.unit_chunks);
      tc::mbar_wait(tempty, tph ^ 1);                  // both epilogues have drained the slots
      tc::fence_after();
      for (int c = c0; c < c1; ++c) {
        tc::mbar_wait(full + stage, phase);
        tc::mbar_wait(pfull + stage, phase);
        tc::fence_after();
        const uint64_t dA = dA0 + (uint64_t)((stage * C::A_BYTES) >> 4);
        const uint64_t dB = dB0 + (uint64_t)((stage * C::B_BYTES) >> 4);
        if (tc::elect_one()) {
          bool started[C::J] = {};
#pragma unroll
          for (int q = 0; q < S; ++q) {
#pragma unroll
            for (int j = 0; j < C::J; ++j) {
              const int p0 = 2 * j - q;                // CTA 0: pair (p0, q) → level 2j
              const bool v0 = p0 >= 0 && 2 * j <= S - 1;
              const bool v1 = p0 + 1 >= 0 && 2 * j + 1 <= S - 1;   // CTA 1: (p0 + 1, q) → level 2j + 1
              if (!v0 && !v1) continue;
              const uint32_t acc = (c > c0 || started[j]) ? 1u : 0u;
              started[j] = true;
              mma_i8_pair(tbase + (uint32_t)(j * TROWS), dA + (uint64_t)(((p0 + 1) * TILE) >> 4),
                          dB + (uint64_t)((q * C::B_HALF) >> 4), IDESC, acc);
            }
          }
          commit_pair(empty + stage);                  // frees the stage in both CTAs
        }
        __syncwarp();
        if (++stage == C::NS) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) commit_pair(tfull);         // this unit's level sums complete, both CTAs
      __syncwarp();
      tph ^= 1;
    }
  } else if (warp >= 2) {                              // ---- epilogue (warps 2..5, both CTAs)
    const int quarter = warp & 3;
    uint32_t tph = 0;
    const uint32_t te0 = peer0(tempty);
    for (int w = cluster; w < items; w += nclusters) {
      const int kq = w / (g.nmb * g.ntn), rem = w % (g.nmb * g.ntn);
      const int mb = rem / g.ntn, tn = rem % g.ntn;
      tc::mbar_wait(tfull, tph);
      tc::fence_after();
      const long row = (long)mb * 128 + quarter * 32 + lane;
      const uint32_t taddr = tbase + ((uint32_t)(quarter * 32) << 16);
      double* wrow = g.ws + (((long)rank * g.nkq + kq) * g.R + row) * g.N;
#pragma unroll 1
      for (int j0 = 0; j0 < TROWS; j0 += 16) {
        uint32_t v[C::J][16];
#pragma unroll
        for (int j = 0; j < C::J; ++j) tc::ld16(taddr + (uint32_t)(j * TROWS + j0), v[j]);
        tc::ld_wait();
        const long col0 = (long)tn * TROWS + j0;
        if (row < g.R && col0 < g.N) {
          double o[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            double acc = 0.0;                          // Σ 2^{-8ℓ} L_ℓ over this CTA's levels, smallest first
#pragma unroll
            for (int j = C::J - 1; j >= 0; --j) {
              const int l = 2 * j + rank;
              if (l <= S - 1) acc = __dadd_rn(acc, __dmul_rn((double)(int)v[j][t], p2m(8 * l)));
            }
            o[t] = acc;
          }
          if (col0 + 16 <= g.N && ((g.N & 1) == 0)) {
#pragma unroll
            for (int t = 0; t < 16; t += 2)
              __stcg(reinterpret_cast<double2*>(wrow + col0 + t), make_double2(o[t], o[t + 1]));
          } else {
#pragma unroll
            for (int t = 0; t < 16; ++t)
              if (col0 + t < g.N) wrow[col0 + t] = o[t];
          }
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) tc::mbar_arrive(tempty);
        else arrive_remote(te0);
      }
      tph ^= 1;
    }
  }
  tc::fence_before();
  tc::cluster_sync();                                  // no CTA leaves while its peer may still signal it
  if (warp == 2) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(C::TMEM_COLS));
  }
}

ENMF_DEV double p2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }   // 2^e, |e| < 1023

// out (R × N, row stride ldo) from the unit partials: Σ_kq ws[kq] + offset corrections per
// level + truncation-bias estimate (ozaki::combine's), scaled by 2^{ea_i + eb_j + 2 − 16}.
template <int S>
__global__ void __launch_bounds__(256) finish(const double* __restrict__ ws, int nparts, long R, long N, long K,
                                              const int* __restrict__ ea, const int* __restrict__ eb,
                                              const int* __restrict__ asum, const int* __restrict__ bsum,
                                              double* __restrict__ out, long ldo, const DevState* st) {
  if (st && !dev_active(st)) return;
  const long i = blockIdx.y;
  const int ei = ea[i];
  int as[S];
#pragma unroll
  for (int p = 0; p < S; ++p) as[p] = asum[(long)p * R + i];
  for (long j = (long)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (long)gridDim.x * blockDim.x) {
    int bs[S];
#pragma unroll
    for (int q = 0; q < S; ++q) bs[q] = bsum[(long)q * N + j];
    const int base = ei + eb[j] + 2;
    // truncation-bias estimate (ozaki::combine): dropped pairs p + q >= S from the digit sums,
    // uncut residuals uniform
    double ra[S], cb[S];
#pragma unroll
    for (int p = 0; p < S; ++p) {
      ra[p] = (double)as[p] + (p ? 128.0 * (double)K : 0.0);
      cb[p] = (double)bs[p] + (p ? 128.0 * (double)K : 0.0);
    }
    double corr = 0.0, sa = 0.0, sb = 0.0;
#pragma unroll
    for (int p = 1; p < S; ++p)
#pragma unroll
      for (int q = S - p; q < S; ++q) corr += (ra[p] * cb[q]) * p2(-8 * (p + q + 2));
    corr /= (double)K;
#pragma unroll
    for (int p = S - 1; p >= 0; --p) {
      sa += ra[p] * p2(-8 * (p + 1));
      sb += cb[p] * p2(-8 * (p + 1));
    }
    corr += (sa + sb) * p2(-8 * S - 1);
    // in units of 2^{base-16}: bias, then the exact offset corrections per level (smallest
    // weight first), then the digit-product partials of the K units in order
    double acc = corr * 65536.0;
#pragma unroll
    for (int l = S - 1; l >= 0; --l) {
      long long cl = 0;
#pragma unroll
      for (int q = 0; q <= l; ++q) {
        const int p = l - q;
        if (q) cl += 128LL * as[p];
        if (p) cl += 128LL * bs[q];
        if (p && q) cl += 16384LL * K;
      }
      acc += (double)cl * p2(-8 * l);
    }
    for (int u = 0; u < nparts; ++u) acc += __ldcs(ws + ((long)u * R + i) * N + j);   // groups × K units, in order
    const int e = base - 16;   // exact power-of-two scaling (ldexp outside the normal range)
    out[i * ldo + j] = (e > -1000 && e < 1000) ? acc * p2(e) : ldexp(acc, e);
  }
}

}  // namespace ozk

// hals_tm.cuh — persistent A-HALS sweep kernel with the iterate held in TENSOR MEMORY
// (nnls.hpp:111-176; default for 64 < r <= 128, i.e. the C5 headline shape).
//
// Same blocked Gauss-Seidel scheme as sweep_ws (hals.cuh): per SM sub-partition a warp
// PAIR — a product warp forming S_b = G[b-rows, :]·H on the FP64 tensor pipe (DMMA.8x8x4)
// and a row warp finishing the 8 rows of block b — handing blocks back and forth, the
// products one block ahead of the row solves (tm_producer_round; scalar FP64 starves next
// to a DMMA stream on the same sub-partition, profiles/r02_share_probe.txt, so only the
// row pass that can hide under the next pair's products runs next to them).  What changes
// is where H lives:
//
//   * H is kept in TMEM, not shared memory.  Each sub-partition owns its 32-lane quarter
//     of the 128 × 512 × 32-bit tensor memory (64 KB): lane = column, two 32-column
//     groups per quarter, row k of a column in 32-bit columns [2k, 2k+1] of its group
//     (group g at TMEM column 2·RMAX·g).  That is 64 columns per sub-partition, 256 per SM:
//     at C5 (32768 columns on 148 SMs = 221 per SM) every column's iterate stays on chip
//     for the whole inner solve — no per-round tile reload, one staging pass per solve.
//   * The product warp reads its B fragments with tcgen05.ld.16x256b: thread (g, t) of the
//     warp receives lane g's 32-bit columns [c + 2t, c + 2t + 1] and lane g + 8's, i.e.
//     H[4s + t][column g] and H[4s + t][column g + 8] — exactly the m8n8k4 B fragment of two
//     8-column tiles (layout checked on the B200: profiles/r02_tmem_probe.txt).  Loads for
//     k-step pair j+1 are in flight while the DMMAs of j issue: 17.7 cycles per DMMA vs
//     20.5 with LDS.128 fragments and 17.4 with B in registers (same probe).
//   * The row warp reads the old rows of a block and writes the new ones with
//     tcgen05.ld/st.32x32b (thread = lane = column), two columns per lane (groups A and B):
//     one hand-off per block covers 64 columns instead of 32, so the latency-bound row
//     chain is paid half as often per column; the two chains interleave.
//   * Shared memory only carries the S hand-off (and the product warp's S_{b+1} partials),
//     and the row-pass constants: 48 KB instead of 141 KB.
//
// Everything else — Gram fragments pre-arranged by ws_prep, the "tail" of the joint
// two-block product, the multiply-free row chain on t = (C − S)/G_kk, the halved gain form,
// the fixed-order grid-wide stall decision (grid_decision) — is sweep_ws's.
#pragma once

#include "hals.cuh"
#include "tc.cuh"

namespace hals {

constexpr int TM_SLD = 40;

// Per-warp phase clock (built only with -DENMF_SWEEP_PROF, tools/gpu_sweep_prof.sh: cycles per
// sweep and phase printed by CTA 0; the product library compiles it away).
struct SwProf {
#ifdef ENMF_SWEEP_PROF
  long long t[8] = {};
  long long last = 0;
  ENMF_DEV void start() { last = clock64(); }
  ENMF_DEV void mark(int i) {
    const long long n = clock64();
    t[i] += n - last;
    last = n;
  }
#else
  ENMF_DEV void start() {}
  ENMF_DEV void mark(int) {}
#endif
};   // S / partial tile row stride (conflict-free 16-byte fragment stores)

// shared memory: Gram fragments (ws_prep order, RMAX² + tails) | S hand-off [pair][group][8][TM_SLD]
// | row-pass constants [NB][48]
template <int RMAX>
__host__ __device__ constexpr int tm_gf_doubles() {
  return RMAX * RMAX + (RMAX / 16) * 64;
}
template <int RMAX>
constexpr int tm_smem_bytes() {
  return (tm_gf_doubles<RMAX>() + 4 * 2 * 8 * TM_SLD + (RMAX / 8) * 48) * 8;
}

// 16 lanes × 256 bits, twice along the columns: thread (g, t) gets lane g's words [c+2t, c+2t+1]
// in v[0..1], lane g+8's in v[2..3], and the same for column c + 8 in v[4..7]
ENMF_DEV void tm_ld_frag(uint32_t ta, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(ta));
}
// 32 lanes × 16 consecutive 32-bit columns (thread i ↔ lane i of this warp's quarter)
ENMF_DEV void tm_ld_rows(uint32_t ta, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(ta));
}
ENMF_DEV void tm_wait_ld16(uint32_t (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}
ENMF_DEV void tm_st_rows(uint32_t ta, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          ta),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
ENMF_DEV void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

ENMF_DEV double tm_d(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }

// tcgen05.wait::ld over the four fragment loads of one k-step pair; it also "rewrites" their
// destination registers, so the compiler cannot read them before the wait
ENMF_DEV void tm_wait_ld32(uint32_t (&f)[4][8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(f[0][0]), "+r"(f[0][1]), "+r"(f[0][2]), "+r"(f[0][3]), "+r"(f[0][4]), "+r"(f[0][5]),
                 "+r"(f[0][6]), "+r"(f[0][7]), "+r"(f[1][0]), "+r"(f[1][1]), "+r"(f[1][2]), "+r"(f[1][3]),
                 "+r"(f[1][4]), "+r"(f[1][5]), "+r"(f[1][6]), "+r"(f[1][7]), "+r"(f[2][0]), "+r"(f[2][1]),
                 "+r"(f[2][2]), "+r"(f[2][3]), "+r"(f[2][4]), "+r"(f[2][5]), "+r"(f[2][6]), "+r"(f[2][7]),
                 "+r"(f[3][0]), "+r"(f[3][1]), "+r"(f[3][2]), "+r"(f[3][3]), "+r"(f[3][4]), "+r"(f[3][5]),
                 "+r"(f[3][6]), "+r"(f[3][7])
               :
               : "memory");
}

// Fragment loads of rows [8j, 8j+8) (k-steps 2j, 2j+1) for the tiles in use: load q covers tiles
// 2q, 2q+1 (q = 0, 1: group A lanes 0-15 / 16-31; q = 2, 3: group B)
template <int NT>
ENMF_DEV void tm_issue(const uint32_t (&la)[4], int j, uint32_t (&f)[4][8]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (2 * q < NT) tm_ld_frag(la[q] + 16 * j, f[q]);
}

// B fragment of tile t, k-step 2j (k = 0) or 2j+1 (k = 1): load t/2, lane half t%2
template <int K>
ENMF_DEV double tm_b(const uint32_t (&f)[4][8], int t) {
  return tm_d(f[t >> 1][4 * K + 2 * (t & 1)], f[t >> 1][4 * K + 2 * (t & 1) + 1]);
}

// c0[t] += A0 · B(t), c1[t] += A1 · B(t) over k-steps 2j, 2j+1; every accumulator's two DMMAs are
// 2·NT instructions apart (≥ 32 cycles > the 26.5-cycle DMMA latency)
template <int NT>
ENMF_DEV void tm_mma_j(double (&c0)[8][2], double (&c1)[8][2], double2 a0, double2 a1, const uint32_t (&f)[4][8]) {
#pragma unroll
  for (int t = 0; t < NT; ++t) dmma884(c0[t][0], c0[t][1], a0.x, tm_b<0>(f, t));
#pragma unroll
  for (int t = 0; t < NT; ++t) dmma884(c1[t][0], c1[t][1], a1.x, tm_b<0>(f, t));
#pragma unroll
  for (int t = 0; t < NT; ++t) dmma884(c0[t][0], c0[t][1], a0.y, tm_b<1>(f, t));
#pragma unroll
  for (int t = 0; t < NT; ++t) dmma884(c1[t][0], c1[t][1], a1.y, tm_b<1>(f, t));
}

// accumulator tiles → the S hand-off rows (tiles 0-3: group A, 4-7: group B)
template <int NT>
ENMF_DEV void tm_store_s(double* Ss, int gi, int gt, const double (&c)[8][2]) {
#pragma unroll
  for (int t = 0; t < NT; ++t)
    *reinterpret_cast<double2*>(Ss + (t >> 2) * 8 * TM_SLD + gi * TM_SLD + (t & 3) * 8 + 2 * gt) =
        make_double2(c[t][0], c[t][1]);
}

// The product warp's part of one round: every tile of the round (both groups) in one pass per
// block pair.  Row blocks in pairs (b, b+1): one pass over H feeds S_b over every row block and
// S_{b+1} over every block but b (whose columns come in as the "tail" once the row warp has solved
// block b; S_{b+1}'s accumulators stay in registers across the hand-off).  Gram fragments stream
// from shared memory (gfs, ws_prep order) next to the TMEM fragment loads, one k-step pair ahead.
// One block of look-ahead: the pass over H starts as soon as S_{b-1} is handed over and takes the
// row blocks in the order b, b+1, ..., b-2 (mod NB) WHILE the row warp solves block b-1 — slowly,
// its scalar FP64 gets one issue slot per ~2 DMMAs next to this stream (profiles/r02_share_probe.txt:
// ~4.7 K cycles per block instead of ~1 K), but hidden under ~8 K cycles of products — and ends with
// block b-1's k-steps once its rows are in.  Block b is then solved with the FP64 pipe to itself
// (nothing to overlap it with: both of the pair's products need its rows).
// abort (speculative decision, nullable): nonzero once the previous sweep was decided to be the
// last — this sweep's rows are discarded, so the round stops at the next block pair; the
// decision is handed to the row warp in *ab_out with the S_b hand-off.  Returns 1 if aborted.
template <int KS, int NB, int NT>
ENMF_DEV int tm_producer_round(uint32_t tq, double* Ss, const double2* gfs, int gi, int gt, int idS, int idH,
                               const volatile int* abort, volatile int* ab_out, SwProf& pf) {
  static_assert(NB == KS / 2 && (NB & (NB - 1)) == 0, "row blocks = k-step pairs, a power of two");
  constexpr uint32_t GC = 8 * KS;   // TMEM columns per group (2 words × RMAX rows)
  const uint32_t la[4] = {tq, tq + (16u << 16), tq + GC, tq + GC + (16u << 16)};
  uint32_t f[2][4][8];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int i = 0; i < 8; ++i) f[0][q][i] = f[1][q][i] = 0u;
#pragma unroll 1
  for (int b = 0; b < NB; b += 2) {
    if (abort) {
      const int ab = *abort;
      if ((threadIdx.x & 31) == 0) *ab_out = ab;
      if (ab) {
        if (b > 0) bar_sync_n<64>(idH);          // the row warp has taken S_{b-1} (one arrival per hand-off)
        bar_arrive_n<64>(idS);                   // the row warp reads the abort and stops too
        return 1;
      }
    }
    double c0[8][2], c1[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) c0[t][0] = c0[t][1] = c1[t][0] = c1[t][1] = 0.0;
    const double2* g0 = gfs + (b * NB) * 32;         // block b's fragments, k-step pair j at j·32
    const double2* g1 = gfs + ((b + 1) * NB) * 32;   // block b+1's (without block b's columns)
    // look-ahead: row blocks b, b+1, ..., b-2 (mod NB) while the row warp still solves block b-1,
    // whose k-steps come last
    tm_issue<NT>(la, b, f[0]);
    double2 a0 = g0[b * 32], a1 = g1[b * 32];
    tm_wait_ld32(f[0]);
#pragma unroll
    for (int jj = 0; jj < NB; ++jj) {
      const int cur = jj & 1;
      const int jn = (b + jj + 1) & (NB - 1);
      double2 n0, n1;
      if (jj + 1 < NB) {
        n0 = g0[jn * 32];
        n1 = g1[jn * 32];
      }
      if (jj + 2 < NB) tm_issue<NT>(la, jn, f[cur ^ 1]);   // next k-step pair in flight while these DMMAs issue
      tm_mma_j<NT>(c0, c1, a0, a1, f[cur]);
      if (jj + 2 == NB) {                        // block b-1: its rows must be final in TMEM
        if (b > 0) {
          pf.mark(0);
          bar_sync_n<64>(idH);
          tc::fence_after();
          pf.mark(2);
        }
        tm_issue<NT>(la, jn, f[cur ^ 1]);
      }
      if (jj + 1 < NB) {
        tm_wait_ld32(f[cur ^ 1]);
        a0 = n0;
        a1 = n1;
      }
    }
    tm_store_s<NT>(Ss, gi, gt, c0);
    pf.mark(0);
    bar_arrive_n<64>(idS);                       // S_b ready (both groups): the row warp solves block b
    const double2 tl = gfs[(16 * KS * KS + (b >> 1) * 64) / 2];
    pf.mark(1);
    bar_sync_n<64>(idH);                         // block b solved
    tc::fence_after();
    pf.mark(2);
    tm_issue<NT>(la, b, f[0]);                   // block b's new rows
    tm_wait_ld32(f[0]);
#pragma unroll
    for (int t = 0; t < NT; ++t) dmma884(c1[t][0], c1[t][1], tl.x, tm_b<0>(f[0], t));
#pragma unroll
    for (int t = 0; t < NT; ++t) dmma884(c1[t][0], c1[t][1], tl.y, tm_b<1>(f[0], t));
    tm_store_s<NT>(Ss, gi, gt, c1);
    bar_arrive_n<64>(idS);                       // S_{b+1} ready
    pf.mark(3);
  }
  return 0;
}

template <int KS, int NB>
ENMF_DEV int tm_producer_round_nt(int nt, uint32_t tq, double* Ss, const double2* gfs, int gi, int gt, int idS,
                                  int idH, const volatile int* abort, volatile int* ab_out, SwProf& pf) {
  switch (nt) {
    case 8: return tm_producer_round<KS, NB, 8>(tq, Ss, gfs, gi, gt, idS, idH, abort, ab_out, pf);
    case 7: return tm_producer_round<KS, NB, 7>(tq, Ss, gfs, gi, gt, idS, idH, abort, ab_out, pf);
    case 6: return tm_producer_round<KS, NB, 6>(tq, Ss, gfs, gi, gt, idS, idH, abort, ab_out, pf);
    case 5: return tm_producer_round<KS, NB, 5>(tq, Ss, gfs, gi, gt, idS, idH, abort, ab_out, pf);
    case 4: return tm_producer_round<KS, NB, 4>(tq, Ss, gfs, gi, gt, idS, idH, abort, ab_out, pf);
    case 3: return tm_producer_round<KS, NB, 3>(tq, Ss, gfs, gi, gt, idS, idH, abort, ab_out, pf);
    case 2: return tm_producer_round<KS, NB, 2>(tq, Ss, gfs, gi, gt, idS, idH, abort, ab_out, pf);
    default: return tm_producer_round<KS, NB, 1>(tq, Ss, gfs, gi, gt, idS, idH, abort, ab_out, pf);
  }
}

// Speculative stall decision (single GPU): the decision on sweep `s` (nnls.hpp:172-173), taken by
// ONE warp of every CTA while the CTA already runs sweep s+1.  Waits until every CTA has published
// its sweep-s gain partial, then forms the total in a fixed order (lane l sums CTAs l, l+32, ...,
// then a fixed xor tree), so every CTA reaches the identical decision; CTA 0 also does the
// solve's bookkeeping (sweep count, first/last gain, sticky non-finite flag, NaN guard).
ENMF_DEV int tm_decide(const Args& a, int s, double& first_total, unsigned bid, unsigned nblk) {
  const int lane = threadIdx.x & 31;
  const unsigned target = (unsigned)(s + 1) * nblk;
  unsigned e;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(e) : "l"(&a.ctl->arrive) : "memory");
  } while (e < target);
  const double* part = a.part + (s & 1) * nblk;
  const int* part_nf = a.part_nf + (s & 1) * nblk;
  double v = 0.0;
  int f = 0;
  for (int b = lane; b < (int)nblk; b += 32) {
    v = __dadd_rn(v, __ldcg(part + b));
    f |= __ldcg(part_nf + b);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  f = __any_sync(0xffffffffu, f) ? 1 : 0;
  if (s == 0) first_total = v;
  const bool stop = (s + 1 >= a.max_sweeps) || (v <= __dmul_rn(a.stall, first_total < 0.0 ? 0.0 : first_total));
  if (bid == 0 && lane == 0) finish_sweep(a, v, f);
  return stop ? 1 : 0;
}

// Copies rows [0, RMAX) of `ncols` columns starting at `col` (lane = column) from global into the
// group at TMEM address tg (zeros outside r × N and past ncols).
template <int RMAX>
ENMF_DEV void tm_stage(uint32_t tg, const double* src, long ld, long col, int ncols, long N, int r, int lane) {
  const bool okc = lane < ncols && col + lane < N;
  const double* sp = src + (okc ? col + lane : 0);
#pragma unroll 2
  for (int k0 = 0; k0 < RMAX; k0 += 8) {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double h = (okc && k0 + i < r) ? sp[(long)(k0 + i) * ld] : 0.0;
      v[2 * i] = (uint32_t)__double2loint(h);
      v[2 * i + 1] = (uint32_t)__double2hiint(h);
    }
    tm_st_rows(tg + 2 * k0, v);
  }
}

// VR (virtual ranks): several ranks' column shards in ONE cooperative launch — CTAs
// [v·vblocks, (v+1)·vblocks) run rank v's solve (its own C / H shard, control block, partial
// buffers and dist::View, a0.vargs[v]), so the sharded path — the synchronous grid decision with
// the cross-rank gain exchange (grid_decision, a.dv) — executes with every rank co-resident on one
// GPU (enmf_gpu_hals_solve_vranks, tests/test_gpu_dist.py).  bid / nblk: this CTA's index and the
// CTA count of its grid, or of its virtual rank's share of the grid.
// (read at the point of use: in the plain kernel they are blockIdx.x / gridDim.x and must not
// occupy registers across the product loops, which run at the register limit)
template <bool VR>
ENMF_DEV unsigned tm_bid(const Args& a0) {
  if constexpr (VR) return blockIdx.x % (unsigned)a0.vblocks;
  else return blockIdx.x;
}
template <bool VR>
ENMF_DEV unsigned tm_nblk(const Args& a0) {
  if constexpr (VR) return (unsigned)a0.vblocks;
  else return gridDim.x;
}

template <int RMAX, bool VR = false>
__global__ void __launch_bounds__(256, 1) sweep_tm(const Args a0, long ntiles) {
  const Args& a = VR ? a0.vargs[blockIdx.x / (unsigned)(VR ? a0.vblocks : 1)] : a0;
  if (VR) ntiles = ((long)a.N + 7) / 8;
#define TM_BID tm_bid<VR>(a0)
#define TM_NBLK tm_nblk<VR>(a0)
  static_assert(RMAX == 128, "two 32-column groups of RMAX rows fill a TMEM lane quarter");
  constexpr int NB = RMAX / 8;
  constexpr int KS = RMAX / 4;
  constexpr uint32_t GC = 2 * RMAX;   // TMEM columns per group
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[256 + 33];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp & 3;
  const bool producer = warp < 4;
  double* Gfs = sm;                                               // Gram fragments (ws_prep order)
  double* Ss = sm + tm_gf_doubles<RMAX>() + pair * (2 * 8 * TM_SLD); // [group][8][TM_SLD]: S hand-off
  // per row block: lower triangle G[8b+l][8b+i] / G_ll (i < l) at l(l-1)/2 + i, G_kk/2 at 28 + l,
  // 1/G_kk at 36 + l (padding rows: unit diagonal)
  double* Gc = sm + tm_gf_doubles<RMAX>() + 4 * 2 * 8 * TM_SLD;
  const int r = a.r;
  {
    const double2* g = reinterpret_cast<const double2*>(a.Gf);
    double2* d = reinterpret_cast<double2*>(Gfs);
    for (int i = threadIdx.x; i < tm_gf_doubles<RMAX>() / 2; i += 256) d[i] = g[i];
  }
  for (int e = threadIdx.x; e < NB * 48; e += 256) {
    const int b = e / 48, j = e % 48;
    double v = 0.0;
    if (j < 28) {
      int l = 1;
      while (l * (l + 1) / 2 <= j) ++l;
      const int i = j - l * (l - 1) / 2, k = 8 * b + l, c = 8 * b + i;
      v = (k < r && c < r) ? __dmul_rn(a.G[(long)k * r + c], __ddiv_rn(1.0, a.G[(long)k * r + k])) : 0.0;
    } else if (j < 44) {
      const int k = 8 * b + ((j - 28) & 7);
      const double d = k < r ? a.G[(long)k * r + k] : 1.0;
      v = j < 36 ? __dmul_rn(0.5, d) : __ddiv_rn(1.0, d);
    }
    Gc[e] = v;
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tq = tmem_base + ((uint32_t)(32 * pair) << 16);   // this pair's lane quarter

  const int idS = 1 + pair, idH = 5 + pair, idP = 9 + pair;
  const long P = (long)TM_NBLK * 4, q = (long)TM_BID * 4 + pair;
  const long tq0 = q * ntiles / P, cnt = (q + 1) * ntiles / P - tq0;
  const int rounds = (int)((cnt + 7) / 8);
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  double gain = 0.0;
  int nf = 0;
  double first_total = 0.0;
  const int gi = lane >> 2, gt = lane & 3;
  const double2* gfs = reinterpret_cast<const double2*>(Gfs) + lane;
  SwProf pf;
  pf.start();
  // Speculative end of sweep (single GPU): sweep s writes its rows to Hb[s & 1] (a.H / a.H2) and
  // publishes its gain partial without waiting; the decision on sweep s is formed during sweep s+1
  // by warp 4 (idle until its first hand-off) and read at the end of sweep s+1.  A "stop" on
  // sweep s discards sweep s+1 — its rows went to the other buffer — and the result is Hb[s & 1].
  // Sharded solves keep the synchronous grid_decision (its cross-GPU exchange).
  const bool spec = a.dv == nullptr && a.H2 != nullptr;
  __shared__ double s_wg[2][4];
  __shared__ int s_wnf[2][4];
  __shared__ int s_dec[2];
  __shared__ int s_abort;                   // the previous sweep was the last (speculative path)
  __shared__ int s_ab[4];                   // per pair: the product warp's abort decision at a pair start
  if (threadIdx.x == 0) s_abort = 0;
  int result_sweep = -1;

  for (int sw = 0;; ++sw) {
    double* const hout = (spec && (sw & 1)) ? a.H2 : a.H;
    if (spec && sw > 0 && warp == 4) {
      const int d = tm_decide(a, sw - 1, first_total, TM_BID, TM_NBLK);
      if (lane == 0) {
        s_dec[(sw - 1) & 1] = d;
        if (d) *(volatile int*)&s_abort = 1;  // stop on sw-1: the rest of sweep sw is discarded
      }
    }
    int aborted = 0;
    for (int i = 0; i < rounds && !aborted; ++i) {
      const long ta = tq0 + (long)i * cnt / rounds;
      const int nt = (int)(tq0 + (long)(i + 1) * cnt / rounds - ta);
      const int ntA = nt < 4 ? nt : 4, ntB = nt - ntA;   // tiles 0-3: group A, 4-7: group B
      const long colA = ta * 8, colB = (ta + ntA) * 8;
      if (!(sw > 0 && rounds == 1)) {            // resident: staged once per solve
        tc::fence_before();
        nb_sync(idP);                            // previous round done with the groups
        tc::fence_after();
        if (producer) tm_stage<RMAX>(tq, src, a.ld, colA, ntA * 8, a.N, r, lane);
        else tm_stage<RMAX>(tq + GC, src, a.ld, colB, ntB * 8, a.N, r, lane);
        tm_wait_st();
        tc::fence_before();
        nb_sync(idP);
        tc::fence_after();
        pf.mark(5);
      }
      if (producer) {
        aborted = tm_producer_round_nt<KS, NB>(nt, tq, Ss, gfs, gi, gt, idS, idH, spec ? &s_abort : nullptr,
                                               &s_ab[pair], pf);
      } else {
        // two columns per lane: cA in group A, cB in group B (predicated, no branches)
        const long ld = a.ld, ld8 = 8 * ld;
        const bool vA = lane < ntA * 8 && colA + lane < a.N;
        const bool vB = lane < ntB * 8 && colB + lane < a.N;
        const double* cpA = a.C + (vA ? colA + lane : 0);
        const double* cpB = a.C + (vB ? colB + lane : 0);
        double* hpA = hout + (vA ? colA + lane : 0);
        double* hpB = hout + (vB ? colB + lane : 0);
        const double* SA = Ss;
        const double* SB = Ss + 8 * TM_SLD;
        double cn[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          cn[i] = (vA && i < r) ? cpA[i * ld] : 0.0;
          cn[8 + i] = (vB && i < r) ? cpB[i * ld] : 0.0;
        }
        uint32_t xa[16], xb[16];
        tm_ld_rows(tq, xa);
        tm_ld_rows(tq + GC, xb);
        int hmax = 0;
        // S slots of lanes past the round's tiles are never written by the product warp: zero them
        // once, so those lanes run t = 0 - 0 (h stays 0, no gain) without a select per row
        if (!(lane < ntA * 8))
#pragma unroll
          for (int i = 0; i < 8; ++i) Ss[i * TM_SLD + lane] = 0.0;
        if (!(lane < ntB * 8))
#pragma unroll
          for (int i = 0; i < 8; ++i) Ss[8 * TM_SLD + i * TM_SLD + lane] = 0.0;
        __syncwarp();
#pragma unroll 1
        for (int b = 0; b < NB; ++b) {
          double bb[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) bb[i] = cn[i];
          if (b + 1 < NB) {
            const double* qa = cpA + ld8;
            const double* qb = cpB + ld8;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              cn[i] = (vA && 8 * (b + 1) + i < r) ? qa[i * ld] : 0.0;
              cn[8 + i] = (vB && 8 * (b + 1) + i < r) ? qb[i * ld] : 0.0;
            }
          }
          double gc[44];
          {
            const double2* gb = reinterpret_cast<const double2*>(Gc + b * 48);
#pragma unroll
            for (int j = 0; j < 22; ++j) {
              const double2 v = gb[j];
              gc[2 * j] = v.x;
              gc[2 * j + 1] = v.y;
            }
          }
          tm_wait_ld16(xa);
          tm_wait_ld16(xb);
          pf.mark(0);
          bar_sync_n<64>(idS);
          pf.mark(1);
          if (spec && !(b & 1) && *(volatile int*)&s_ab[pair]) {   // sweep discarded (see tm_producer_round)
            aborted = 1;
            break;
          }
          double x[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            // t = C/G_kk - S/G_kk (the Gram fragments are pre-divided by G_kk, ws_prep SCALE)
            const double sa = fma(bb[i], gc[36 + i], -SA[i * TM_SLD + lane]);
            const double sb = fma(bb[8 + i], gc[36 + i], -SB[i * TM_SLD + lane]);
            bb[i] = sa;
            bb[8 + i] = sb;
            x[i] = tm_d(xa[2 * i], xa[2 * i + 1]);
            x[8 + i] = tm_d(xb[2 * i], xb[2 * i + 1]);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double h0 = pos_part_ws(bb[i]);
            const double h1 = pos_part_ws(bb[8 + i]);
#pragma unroll
            for (int l = i + 1; l < 8; ++l) {
              bb[l] = fma(-gc[l * (l - 1) / 2 + i], h0, bb[l]);
              bb[8 + l] = fma(-gc[l * (l - 1) / 2 + i], h1, bb[8 + l]);
            }
            // G_kk((x-t)² - (h-t)²) = (x-h)·(G_kk/2)·(x+h-2t)·2, accumulated halved (an integer-pipe
            // max(-t, 0) in place of x+h costs more issue slots than the DADD it saves: measured)
            const double u0 = __dsub_rn(x[i], h0), u1 = __dsub_rn(x[8 + i], h1);
            gain = fma(__dmul_rn(u0, gc[28 + i]), fma(-2.0, bb[i], __dadd_rn(x[i], h0)), gain);
            gain = fma(__dmul_rn(u1, gc[28 + i]), fma(-2.0, bb[8 + i], __dadd_rn(x[8 + i], h1)), gain);
            x[i] = h0;
            x[8 + i] = h1;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            xa[2 * i] = (uint32_t)__double2loint(x[i]);
            xa[2 * i + 1] = (uint32_t)__double2hiint(x[i]);
            xb[2 * i] = (uint32_t)__double2loint(x[8 + i]);
            xb[2 * i + 1] = (uint32_t)__double2hiint(x[8 + i]);
          }
          tm_st_rows(tq + 16 * b, xa);
          tm_st_rows(tq + GC + 16 * b, xb);
          tm_wait_st();
          tc::fence_before();
          if (b + 1 < NB) bar_arrive_n<64>(idH);
          pf.mark(2);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (vA && 8 * b + i < r) hpA[i * ld] = x[i];
            if (vB && 8 * b + i < r) hpB[i * ld] = x[8 + i];
            hmax = max(hmax, max(__double2hiint(x[i]), __double2hiint(x[8 + i])));
          }
          if (b + 1 < NB) {                      // old rows of the next block (in flight over the hand-off)
            tm_ld_rows(tq + 16 * (b + 1), xa);
            tm_ld_rows(tq + GC + 16 * (b + 1), xb);
          }
          cpA += ld8;
          cpB += ld8;
          hpA += ld8;
          hpB += ld8;
          pf.mark(3);
        }
        nf |= hmax >= 0x7FF00000;
      }
    }
    if (spec) {
      // ---- speculative end of sweep `sw` ----
      if (!producer) {
        double g = __dadd_rn(gain, gain);   // gains are accumulated halved
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) g = __dadd_rn(g, __shfl_xor_sync(0xffffffffu, g, off));
        const int f = __any_sync(0xffffffffu, nf) ? 1 : 0;
        if (lane == 0) {
          s_wg[sw & 1][pair] = g;
          s_wnf[sw & 1][pair] = f;
        }
      }
      tc::fence_before();                    // the row warps' last TMEM stores before the next sweep
      pf.mark(6);
      __syncthreads();
      tc::fence_after();
      const int last = sw + 1 >= a.max_sweeps;
      if (warp == 4 && lane == 0) {          // this CTA's sweep-sw partial (fixed order over the warps)
        const double g = __dadd_rn(__dadd_rn(s_wg[sw & 1][0], s_wg[sw & 1][1]),
                                   __dadd_rn(s_wg[sw & 1][2], s_wg[sw & 1][3]));
        const int f = s_wnf[sw & 1][0] | s_wnf[sw & 1][1] | s_wnf[sw & 1][2] | s_wnf[sw & 1][3];
        a.part[(sw & 1) * TM_NBLK + TM_BID] = g;
        a.part_nf[(sw & 1) * TM_NBLK + TM_BID] = f;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(&a.ctl->arrive) : "memory");
      }
      pf.mark(4);
      if (sw > 0 && s_dec[(sw - 1) & 1]) {   // sweep sw-1 was the last: sweep sw is discarded
        result_sweep = sw - 1;
        break;
      }
      if (last) {                            // max_sweeps reached: no speculation past the cap
        if (TM_BID == 0 && warp == 4) tm_decide(a, sw, first_total, TM_BID, TM_NBLK);   // bookkeeping only
        result_sweep = sw;
        break;
      }
      gain = 0.0;
      nf = 0;
      src = hout;
      continue;
    }
    // ---- grid-wide end of sweep `sw` (the row warps' last TMEM stores are ordered before the
    // next sweep's fragment loads by the fences around grid_decision's block barriers) ----
    tc::fence_before();
    pf.mark(6);
    const int cont = grid_decision(a, gain, nf, sw, first_total, red, TM_BID, TM_NBLK);
    tc::fence_after();
    pf.mark(4);
    if (!cont) {
      result_sweep = sw;
      break;
    }
    gain = 0.0;
    nf = 0;
    src = a.H;
  }
#ifdef ENMF_SWEEP_PROF
  if ((TM_BID == 0 || TM_BID == TM_NBLK / 2) && lane == 0)
    printf("sweep_tm prof cta %d warp %d sweeps %d cycles/sweep: %lld %lld %lld %lld | decision %lld | stage %lld | "
           "end %lld\n", TM_BID, warp, result_sweep + 1, pf.t[0] / (result_sweep + 1), pf.t[1] / (result_sweep + 1),
           pf.t[2] / (result_sweep + 1), pf.t[3] / (result_sweep + 1), pf.t[4] / (result_sweep + 1),
           pf.t[5] / (result_sweep + 1), pf.t[6] / (result_sweep + 1));
#endif
  if (spec && (result_sweep & 1)) {
    // the result is in the scratch buffer: copy this pair's columns into a.H (rows < r)
    const long c0 = tq0 * 8, c1 = min((tq0 + cnt) * 8, (long)a.N);
    const int t = (threadIdx.x & 31) + (producer ? 0 : 32);
    for (long col = c0 + t; col < c1; col += 64)
      for (int k = 0; k < r; ++k) a.H[(long)k * a.ld + col] = a.H2[(long)k * a.ld + col];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}


#undef TM_BID
#undef TM_NBLK

}  // namespace hals

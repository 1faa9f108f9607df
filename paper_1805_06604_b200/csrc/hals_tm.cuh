// hals_tm.cuh — persistent A-HALS sweep kernel with the iterate held in TENSOR MEMORY
// (nnls.hpp:111-176; default for 64 < r <= 128, i.e. the C5 headline shape).
//
// Same blocked Gauss-Seidel scheme as sweep_ws (hals.cuh): per SM sub-partition a warp
// PAIR — a product warp forming S_b = G[b-rows, :]·H on the FP64 tensor pipe (DMMA.8x8x4)
// and a row warp finishing the 8 rows of block b one column per lane — strictly
// alternating, because scalar FP64 starves next to a DMMA stream on the same
// sub-partition (profiles/r01_xsmsp_probe.txt).  What changes is where H lives:
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
// two-block product, the multiply-free row chain t = (C − S)/G_kk, the halved gain form,
// the fixed-order grid-wide stall decision (grid_decision) — is sweep_ws's.
#pragma once

#include "hals.cuh"
#include "tc.cuh"

namespace hals {

constexpr int TM_SLD = 40;   // S / partial tile row stride (conflict-free 16-byte fragment stores)

template <int RMAX>
constexpr int tm_smem_bytes() {
  return (2 * 4 * 2 * 8 * TM_SLD + (RMAX / 8) * 48) * 8;
}

// 16 lanes × 256 bits, twice along the columns: thread (g, t) gets lane g's words [c+2t, c+2t+1]
// in v[0..1], lane g+8's in v[2..3], and the same for column c + 8 in v[4..7]
ENMF_DEV void tm_ld_frag(uint32_t ta, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(ta));
}
// tcgen05.wait::ld that also "rewrites" the destination registers of the loads it waits for, so
// the compiler cannot read them before the wait
ENMF_DEV void tm_wait_ld8(uint32_t (&u)[8], uint32_t (&w)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(u[0]), "+r"(u[1]), "+r"(u[2]), "+r"(u[3]), "+r"(u[4]), "+r"(u[5]), "+r"(u[6]), "+r"(u[7]),
                 "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]), "+r"(w[7])
               :
               : "memory");
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

// B fragments of k-steps (2j, 2j+1) for tiles 0..3 from the two 16-lane loads (see ws_mma2's p[])
ENMF_DEV void tm_frags(const uint32_t (&u)[8], const uint32_t (&w)[8], double2 (&p)[4]) {
  p[0] = make_double2(tm_d(u[0], u[1]), tm_d(u[2], u[3]));
  p[2] = make_double2(tm_d(u[4], u[5]), tm_d(u[6], u[7]));
  p[1] = make_double2(tm_d(w[0], w[1]), tm_d(w[2], w[3]));
  p[3] = make_double2(tm_d(w[4], w[5]), tm_d(w[6], w[7]));
}

// One group's joint two-block product: acc0 = S_b, acc1 = S_{b+1} without block b's columns;
// tg = TMEM address of the group (this warp's lane quarter, column 0 of the group).
template <int KS, int NT>
ENMF_DEV void tm_products(uint32_t tg, const double (&A0)[KS], const double (&A1)[KS], double* Sg, double* Pg, int gi,
                          int gt) {
  double acc0[4][2], acc1[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) acc0[t][0] = acc0[t][1] = acc1[t][0] = acc1[t][1] = 0.0;
  uint32_t u[2][8], w[2][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[0][i] = w[1][i] = 0u;
  tm_ld_frag(tg, u[0]);
  if (NT > 2) tm_ld_frag(tg + (16u << 16), w[0]);
  tm_wait_ld8(u[0], w[0]);
#pragma unroll
  for (int j = 0; j < KS / 2; ++j) {
    const int c = j & 1;
    if (j + 1 < KS / 2) {           // next k-step pair in flight while this one's DMMAs issue
      tm_ld_frag(tg + 16 * (j + 1), u[c ^ 1]);
      if (NT > 2) tm_ld_frag(tg + (16u << 16) + 16 * (j + 1), w[c ^ 1]);
    }
    double2 p[4];
    tm_frags(u[c], w[c], p);
    ws_mma2<NT>(acc0, A0[2 * j], A0[2 * j + 1], p);
    ws_mma2<NT>(acc1, A1[2 * j], A1[2 * j + 1], p);
    if (j + 1 < KS / 2) tm_wait_ld8(u[c ^ 1], w[c ^ 1]);
  }
  ws_store_s(Sg, gi, gt, acc0);
  ws_store_s(Pg, gi, gt, acc1);
}

// S_{b+1} += G[b+1 rows, block b columns] · (block b's new rows); partial from Pg, result to Sg
template <int NT>
ENMF_DEV void tm_tail(uint32_t tg, int b, double2 tl, double* Sg, const double* Pg, int gi, int gt) {
  uint32_t u[8], w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = 0u;
  tm_ld_frag(tg + 16 * b, u);
  if (NT > 2) tm_ld_frag(tg + (16u << 16) + 16 * b, w);
  double acc[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const double2 v = *reinterpret_cast<const double2*>(Pg + gi * TM_SLD + t * 8 + 2 * gt);
    acc[t][0] = v.x;
    acc[t][1] = v.y;
  }
  tm_wait_ld8(u, w);
  double2 p[4];
  tm_frags(u, w, p);
  ws_mma2<NT>(acc, tl.x, tl.y, p);
  ws_store_s(Sg, gi, gt, acc);
}

template <int KS>
ENMF_DEV void tm_products_nt(int nt, uint32_t tg, const double (&A0)[KS], const double (&A1)[KS], double* Sg,
                             double* Pg, int gi, int gt) {
  switch (nt) {
    case 4: tm_products<KS, 4>(tg, A0, A1, Sg, Pg, gi, gt); break;
    case 3: tm_products<KS, 3>(tg, A0, A1, Sg, Pg, gi, gt); break;
    case 2: tm_products<KS, 2>(tg, A0, A1, Sg, Pg, gi, gt); break;
    default: tm_products<KS, 1>(tg, A0, A1, Sg, Pg, gi, gt); break;
  }
}
ENMF_DEV void tm_tail_nt(int nt, uint32_t tg, int b, double2 tl, double* Sg, const double* Pg, int gi, int gt) {
  switch (nt) {
    case 4: tm_tail<4>(tg, b, tl, Sg, Pg, gi, gt); break;
    case 3: tm_tail<3>(tg, b, tl, Sg, Pg, gi, gt); break;
    case 2: tm_tail<2>(tg, b, tl, Sg, Pg, gi, gt); break;
    default: tm_tail<1>(tg, b, tl, Sg, Pg, gi, gt); break;
  }
}

// The product warp's part of one round (groups A and B of this sub-partition).
template <int KS, int NB>
ENMF_DEV void tm_producer_round(uint32_t tq, int ntA, int ntB, double* Ss, double* Ps, const double2* gf, int gi,
                                int gt, int idS, int idH) {
  constexpr uint32_t GC = 8 * KS;   // TMEM columns per group (2 words × RMAX rows)
  double A0[KS], A1[KS];
#pragma unroll
  for (int s = 0; s < KS; s += 2) {
    const double2 f0 = gf[(s / 2) * 32];
    const double2 f1 = gf[(KS / 2 + s / 2) * 32];
    A0[s] = f0.x; A0[s + 1] = f0.y;
    A1[s] = f1.x; A1[s + 1] = f1.y;
  }
  double* SA = Ss;
  double* SB = Ss + 8 * TM_SLD;
  double* PA = Ps;
  double* PB = Ps + 8 * TM_SLD;
#pragma unroll 1
  for (int b = 0; b < NB; b += 2) {
    if (b > 0) {
      bar_sync_n<64>(idH);                       // rows of block b-1 are final in TMEM
      tc::fence_after();
    }
    tm_products_nt<KS>(ntA, tq, A0, A1, SA, PA, gi, gt);
    if (ntB > 0) tm_products_nt<KS>(ntB, tq + GC, A0, A1, SB, PB, gi, gt);
    bar_arrive_n<64>(idS);                       // S_b ready (both groups): the row warp solves block b
    // while it does: this pair's tail fragments and the next pair's Gram fragments
    const double2 tl = gf[(16 * KS * KS + (b >> 1) * 64) / 2];
    if (b + 2 < NB) {
#pragma unroll
      for (int s = 0; s < KS; s += 2) {
        const double2 f0 = gf[(((b + 2) * KS / 2) + s / 2) * 32];
        const double2 f1 = gf[(((b + 3) * KS / 2) + s / 2) * 32];
        A0[s] = f0.x; A0[s + 1] = f0.y;
        A1[s] = f1.x; A1[s + 1] = f1.y;
      }
    }
    bar_sync_n<64>(idH);                         // block b solved
    tc::fence_after();
    tm_tail_nt(ntA, tq, b, tl, SA, PA, gi, gt);
    if (ntB > 0) tm_tail_nt(ntB, tq + GC, b, tl, SB, PB, gi, gt);
    bar_arrive_n<64>(idS);                       // S_{b+1} ready
  }
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

template <int RMAX>
__global__ void __launch_bounds__(256, 1) sweep_tm(Args a, long ntiles) {
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
  double* Ss = sm + pair * (2 * 8 * TM_SLD);                      // [group][8][TM_SLD]: S hand-off
  double* Ps = sm + 4 * 2 * 8 * TM_SLD + pair * (2 * 8 * TM_SLD);  // product warp's S_{b+1} partials
  // per row block: lower triangle G[8b+l][8b+i] / G_ll (i < l) at l(l-1)/2 + i, G_kk/2 at 28 + l,
  // 1/G_kk at 36 + l (padding rows: unit diagonal)
  double* Gc = sm + 2 * 4 * 2 * 8 * TM_SLD;
  const int r = a.r;
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
  const long P = (long)gridDim.x * 4, q = (long)blockIdx.x * 4 + pair;
  const long tq0 = q * ntiles / P, cnt = (q + 1) * ntiles / P - tq0;
  const int rounds = (int)((cnt + 7) / 8);
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  double gain = 0.0;
  int nf = 0;
  double first_total = 0.0;
  const int gi = lane >> 2, gt = lane & 3;
  const double2* gf = reinterpret_cast<const double2*>(a.Gf) + lane;

  for (int sw = 0;; ++sw) {
    for (int i = 0; i < rounds; ++i) {
      const long ta = tq0 + (long)i * cnt / rounds;
      const int nt = (int)(tq0 + (long)(i + 1) * cnt / rounds - ta);
      const int ntA = (nt + 1) / 2, ntB = nt - ntA;
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
      }
      if (producer) {
        tm_producer_round<KS, NB>(tq, ntA, ntB, Ss, Ps, gf, gi, gt, idS, idH);
      } else {
        // two columns per lane: cA in group A, cB in group B (predicated, no branches)
        const long ld = a.ld, ld8 = 8 * ld;
        const bool vA = lane < ntA * 8 && colA + lane < a.N;
        const bool vB = lane < ntB * 8 && colB + lane < a.N;
        const double* cpA = a.C + (vA ? colA + lane : 0);
        const double* cpB = a.C + (vB ? colB + lane : 0);
        double* hpA = a.H + (vA ? colA + lane : 0);
        double* hpB = a.H + (vB ? colB + lane : 0);
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
          bar_sync_n<64>(idS);
          double x[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            bb[i] = __dmul_rn(__dsub_rn(bb[i], SA[i * TM_SLD + lane]), gc[36 + i]);
            bb[8 + i] = __dmul_rn(__dsub_rn(bb[8 + i], SB[i * TM_SLD + lane]), gc[36 + i]);
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
            const double u0 = __dsub_rn(x[i], h0), v0 = __dadd_rn(x[i], h0);
            const double u1 = __dsub_rn(x[8 + i], h1), v1 = __dadd_rn(x[8 + i], h1);
            gain = fma(__dmul_rn(u0, gc[28 + i]), fma(-2.0, bb[i], v0), gain);
            gain = fma(__dmul_rn(u1, gc[28 + i]), fma(-2.0, bb[8 + i], v1), gain);
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
        }
        nf |= hmax >= 0x7FF00000;
      }
    }
    // ---- grid-wide end of sweep `sw` (the row warps' last TMEM stores are ordered before the
    // next sweep's fragment loads by the fences around grid_decision's block barriers) ----
    tc::fence_before();
    const int cont = grid_decision(a, gain, nf, sw, first_total, red);
    tc::fence_after();
    if (!cont) break;
    gain = 0.0;
    nf = 0;
    src = a.H;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace hals

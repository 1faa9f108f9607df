// hals.cuh — multi-sweep A-HALS inner solver (nnls.hpp:111-176) on sm_100a.
//
// One launch = one Gauss-Seidel sweep over all r rows for every right-hand
// side (column).  Columns are independent within a sweep; the
// only coupling is the global stall rule
//     stop if sweep >= max_sweeps  or  gain <= stall_fraction * max(first_gain, 0)
// (nnls.hpp:172-173), evaluated by the last block to finish (fixed-order sum
// of per-block gains -> deterministic) which also drives the CUDA-graph
// conditional WHILE node that repeats the sweep kernel.
//
// Fast kernel: TPC threads per column, each holding S rows of that column in
// registers (row j lives in thread j % TPC, slot j / TPC); the r×r Gram sits
// in shared memory with its diagonal zeroed and permuted so each thread
// streams its own slots with 16-byte broadcast loads.  Per row k:
//     dot = sum_{j != k} G[k][j] h[j]     (4 FMA chains, then xor-shuffle over TPC)
//     target = (C[k][t] - dot) / G[k][k];  h[k] = max(target, 0)
//     gain += G[k][k] * ((h_old - target)^2 - (h_new - target)^2)
// Exact kernel (precision = FP64_EXACT, and the generic path for r > 128):
// one thread per column in the reference's order (j ascending, gkj == 0
// skipped, no FMA) and a second kernel that sums the per-row gains over the
// columns in the reference's sequential order, so the sweep count and the
// iterates are bitwise those of hals_solve.
#pragma once

#include "common.cuh"
#include "dist.cuh"

namespace hals {

constexpr int NT = 256;

struct Args {
  const double* G;        // r×r
  const double* C;        // r×N, row stride ld
  const double* Hin;      // warm start (read by sweep 1 only)
  double* H;              // r×N output / in-place iterate
  long ld;
  int r, N;
  int max_sweeps;
  double stall;
  HalsCtl* ctl;
  double* part;           // per-block gain partials
  int* part_nf;           // per-block non-finite flags
  double* terms;          // exact kernel: r×N per-row gain terms
  DevState* st;           // nullable
  int side;               // 0: H update, 1: W update (error message / flags)
  unsigned long long cond;  // cudaGraphConditionalHandle (0 = none)
  int use_cond;
  const dist::View* dv;     // multi-GPU: all-reduce the sweep gain across ranks (nullable)
  const double* Gf;         // sweep_ws: Gram in A-fragment order (ws_prep)
  double* H2;               // sweep_tm: r×N scratch (row stride ld) for odd sweeps (speculative stall decision)
  // virtual ranks (sweep_tm<128, true>, one cooperative launch over several ranks' column shards — the
  // on-device check of the sharded sweep path, enmf_gpu_hals_solve_vranks): rank v's arguments
  // and the CTAs per rank
  const Args* vargs;
  int vblocks;
};

ENMF_DEV void set_cond(const Args& a, unsigned v) {
  if (a.use_cond) cudaGraphSetConditional((cudaGraphConditionalHandle)a.cond, v);
}

// Stall rule + bookkeeping after a sweep whose total gain is `gain`.
ENMF_DEV void finish_sweep(const Args& a, double gain, int nonfinite) {
  HalsCtl* c = a.ctl;
  const int s = c->sweeps + 1;
  c->sweeps = s;
  if (s == 1) c->first_gain = gain;
  c->last_gain = gain;
  const double fg = c->first_gain;
  const bool stop = (s >= a.max_sweeps) || (gain <= __dmul_rn(a.stall, fg < 0.0 ? 0.0 : fg));
  c->cont = stop ? 0 : 1;
  // sticky over the sweeps of a solve: the block products form 0·h for the zeroed Gram entries
  // the reference skips (nnls.hpp:121, gkj == 0), so an overflowed row (+inf) turns into NaN and
  // then 0 in the next sweep instead of staying +inf as in the reference
  c->nonfinite |= nonfinite;
  if (stop && c->nonfinite && a.st) {
    // NaN guard on the finished iterate (engine.hpp:334-337 / 380-383)
    if (a.st->active) {
      a.st->error_code = ENMF_NON_FINITE;
      a.st->active = 0;
    }
  }
  __threadfence();
  set_cond(a, stop ? 0u : 1u);
}

// Returns true (uniformly) if this launch must do no work.
ENMF_DEV bool sweep_skipped(const Args& a) {
  const bool skip = (a.st && !dev_active(a.st)) || !*(volatile int*)&a.ctl->cont;
  if (skip && blockIdx.x == 0 && threadIdx.x == 0) set_cond(a, 0u);
  return skip;
}

// Last-arriving block: fixed-order sum of the per-block partials.
template <int NTH>
ENMF_DEV void last_block_reduce_n(const Args& a, double block_gain, int block_nf, double* red) {
  __shared__ unsigned s_last;
  if (threadIdx.x == 0) {
    a.part[blockIdx.x] = block_gain;
    a.part_nf[blockIdx.x] = block_nf;
    __threadfence();
    const unsigned prev = atomicAdd(&a.ctl->arrive, 1u);
    s_last = (prev == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double v = 0.0;
  int nf = 0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += NTH) {
    v = __dadd_rn(v, __ldcg(a.part + b));
    nf |= __ldcg(a.part_nf + b);
  }
  double total = block_reduce_sum_any(v, red);
  nf = __syncthreads_or(nf);
  if (threadIdx.x == 0) {
    a.ctl->arrive = 0;
    if (a.dv) dist::allreduce_gain(*a.dv, total, nf, &total, &nf);  // global stall rule
    finish_sweep(a, total, nf);
  }
}

template <int S, int TPC>
constexpr int smem_bytes() {
  return (S * TPC) * TPC * (S + 2) * 8 + (S * TPC) * 8;
}

template <int S, int TPC>
__global__ void __launch_bounds__(NT) sweep_fast(Args a) {
  constexpr int RMAX = S * TPC;
  constexpr int GROW = TPC * (S + 2);
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  double* Gs = sm;                 // [RMAX][TPC][S+2], diagonal zeroed
  double* Gd = sm + RMAX * GROW;   // diag
  __shared__ double red[NT];

  const int r = a.r;
  for (int e = threadIdx.x; e < RMAX * TPC * S; e += NT) {
    const int k = e / (TPC * S), rem = e % (TPC * S), q = rem / S, s = rem % S;
    const int j = s * TPC + q;
    double v = 0.0;
    if (k < r && j < r && j != k) v = a.G[k * r + j];
    Gs[k * GROW + q * (S + 2) + s] = v;
  }
  for (int k = threadIdx.x; k < RMAX; k += NT) Gd[k] = k < r ? a.G[k * r + k] : 1.0;
  __syncthreads();

  const int q = threadIdx.x % TPC;
  const int t = blockIdx.x * (NT / TPC) + threadIdx.x / TPC;
  const bool valid = t < a.N;
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;

  double h[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int j = s * TPC + q;
    h[s] = (valid && j < r) ? src[(long)j * a.ld + t] : 0.0;
  }
  double gain = 0.0;
  double cnext = (valid) ? a.C[t] : 0.0;
  // Rows k >= r are padding: zero Gram row, unit diagonal, zero cross term,
  // so their update is a no-op (target 0, h stays 0, gain 0); no data-dependent
  // exit keeps the loop fully unrolled and every h[] index static.
#pragma unroll
  for (int k = 0; k < RMAX; ++k) {
    const double ck = cnext;
    if (k + 1 < r && valid) cnext = a.C[(long)(k + 1) * a.ld + t];
    else cnext = 0.0;
    const double2* gk = reinterpret_cast<const double2*>(Gs + k * GROW + q * (S + 2));
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int s2 = 0; s2 < S / 2; ++s2) {
      const double2 gv = gk[s2];
      acc[(2 * s2) & 3] = fma(gv.x, h[2 * s2], acc[(2 * s2) & 3]);
      acc[(2 * s2 + 1) & 3] = fma(gv.y, h[2 * s2 + 1], acc[(2 * s2 + 1) & 3]);
    }
    double dot = __dadd_rn(__dadd_rn(acc[0], acc[1]), __dadd_rn(acc[2], acc[3]));
#pragma unroll
    for (int off = 1; off < TPC; off <<= 1) dot = __dadd_rn(dot, __shfl_xor_sync(0xffffffffu, dot, off));
    const double gkk = Gd[k];
    const double target = __ddiv_rn(__dsub_rn(ck, dot), gkk);
    const double next = target > 0.0 ? target : 0.0;
    if (q == (k % TPC)) {
      const double d_old = __dsub_rn(h[k / TPC], target);
      const double d_new = __dsub_rn(next, target);
      gain = fma(gkk, __dsub_rn(__dmul_rn(d_old, d_old), __dmul_rn(d_new, d_new)), gain);
      h[k / TPC] = next;
    }
  }
  int nf = 0;
  if (valid) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int j = s * TPC + q;
      if (j < r) {
        a.H[(long)j * a.ld + t] = h[s];
        nf |= !isfinite(h[s]);
      }
    }
  }
  const double bg = block_reduce_sum<NT>(valid ? gain : 0.0, red);
  nf = __syncthreads_or(nf);
  last_block_reduce_n<NT>(a, bg, nf, red);
}

// ---- paired-warp tensor-core sweep (default) ----------------------------------
//
// Every SM sub-partition runs one PAIR of warps over its own 32 columns:
//   * the product warp issues the DMMAs of the block products
//         S_b = G[b-rows, :] · H        (A = Gram fragment in registers, B = H in smem)
//   * the row warp owns one column per lane and finishes the 8 rows of block b
//     sequentially (nnls.hpp:117-148 per row), entirely in registers, writing the
//     new rows straight into the H tile.
// The two phases strictly alternate (named-barrier hand-offs, bar.arrive by the
// producer of a tile, bar.sync by its consumer): measured on B200
// (tools/probe/pipe_probe.cu, profiles/r01_latency_probes.txt), scalar FP64
// instructions on a sub-partition whose DMMA pipe is streaming are starved
// (~75 cycles per independent op, ~500 per dependent op), so the row chain runs
// while the sub-partition's DMMA pipe is idle and takes ~0.3 K cycles instead of
// ~1.7 K when overlapped.  Diagonal blocks enter the DMMA with their lower triangle
// (diagonal included) zeroed, so the row warp only subtracts
// sum_{j<k in block} G_kj h_new_j.
//
// Gram fragments come pre-arranged by ws_prep (once per inner solve): Gf holds,
// for row block b and k-step pair s2, the two A-fragment values of every lane
// contiguously, so a lane fetches two k-steps with one 16-byte load, and the
// fragments of block b+1 stream into the registers freed by block b.  The H tile
// is stored with 16-byte chunks holding columns (c, c+8) and an XOR swizzle per
// row, so each lane reads the B fragments of its 4 column tiles with two
// conflict-free 16-byte loads per k-step.
constexpr int WS_SLD = 40;   // S tile row stride: conflict-free 16-byte fragment stores

template <int RMAX>
constexpr int ws_smem_bytes() {
  return (4 * (RMAX * 32 + 8 * WS_SLD) + (RMAX / 8) * 48) * 8;
}

// position of (row k, column c) in a swizzled 32-column tile
ENMF_DEV int ws_pos(int k, int c) {
  const int sw = ((k & 1) << 2) | ((k >> 1) & 1);
  return k * 32 + 2 * ((2 * (c & 7) + (c >> 4)) ^ sw) + ((c >> 3) & 1);
}

ENMF_DEV void nb_sync(int id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory"); }
ENMF_DEV void nb_arrive(int id) { asm volatile("bar.arrive %0, 64;\n" ::"r"(id) : "memory"); }

ENMF_DEV double pos_part_ws(double t) {
  const long long b = __double_as_longlong(t);
  return (b > 0 && b <= 0x7FF0000000000000LL) ? t : 0.0;   // t > 0 (NaN -> 0, as `t > 0 ? t : 0`)
}

// Gf[((b·KS/2 + s2)·32 + lane)·2 + e] = G[8b + lane/4][4(2·s2+e) + lane%4], zero outside r×r,
// on/below the diagonal inside diagonal blocks, and — for odd b — in the columns of block
// b-1, whose fragments go to Gf[RMAX² + ...] instead (the "tail" of the paired product).
// SPLIT = false (sweep_t2): no tail split, every block's fragments in the main array.
// SCALE (sweep_tm): row k divided by G_kk, so the block products come out as S/G_kk and the row
// pass forms t = C/G_kk - S/G_kk with one fma.
template <int RMAX, bool SPLIT = true, bool SCALE = false>
__global__ void ws_prep(const double* G, int r, double* Gf, const DevState* st, const HalsCtl* ctl) {
  if ((st && !dev_active(st)) || !ctl->cont) return;
  constexpr int KS = RMAX / 4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < RMAX * RMAX; i += gridDim.x * blockDim.x) {
    const int e = i & 1, lane = (i >> 1) & 31, s2 = (i >> 6) % (KS / 2), b = (i >> 6) / (KS / 2);
    const int s = 2 * s2 + e, gi = lane >> 2, gt = lane & 3;
    const int row = 8 * b + gi, col = 4 * s + gt;
    double v = 0.0;
    if (row < r && col < r && !((s >> 1) == b && col - 8 * b <= gi)) {
      v = G[(long)row * r + col];
      if (SCALE) v = __dmul_rn(v, __ddiv_rn(1.0, G[(long)row * r + row]));
    }
    const bool tail = SPLIT && (b & 1) && s2 == b - 1;
    Gf[i] = tail ? 0.0 : v;
    if (tail) Gf[RMAX * RMAX + (b >> 1) * 64 + lane * 2 + e] = v;
  }
}

// B fragments of k-steps (2j, 2j+1) — rows 8j..8j+7 — for the NT column tiles of a pair
template <int NT>
ENMF_DEV void ws_ldb(const double* Hs, int j, int gt, int bx0, int bx1, double2 (&p)[4]) {
  const int k0 = 8 * j + gt, k1 = k0 + 4;
  p[0] = *reinterpret_cast<const double2*>(Hs + k0 * 32 + bx0);
  if (NT > 2) p[1] = *reinterpret_cast<const double2*>(Hs + k0 * 32 + bx1);
  p[2] = *reinterpret_cast<const double2*>(Hs + k1 * 32 + bx0);
  if (NT > 2) p[3] = *reinterpret_cast<const double2*>(Hs + k1 * 32 + bx1);
}

// acc[t] += a0 · B(k-step 2j) + a1 · B(k-step 2j+1) for the NT tiles
template <int NT>
ENMF_DEV void ws_mma2(double (&acc)[4][2], double a0, double a1, const double2 (&p)[4]) {
  dmma884(acc[0][0], acc[0][1], a0, p[0].x);
  if (NT > 1) dmma884(acc[1][0], acc[1][1], a0, p[0].y);
  if (NT > 2) dmma884(acc[2][0], acc[2][1], a0, p[1].x);
  if (NT > 3) dmma884(acc[3][0], acc[3][1], a0, p[1].y);
  dmma884(acc[0][0], acc[0][1], a1, p[2].x);
  if (NT > 1) dmma884(acc[1][0], acc[1][1], a1, p[2].y);
  if (NT > 2) dmma884(acc[2][0], acc[2][1], a1, p[3].x);
  if (NT > 3) dmma884(acc[3][0], acc[3][1], a1, p[3].y);
}

ENMF_DEV void ws_store_s(double* Ss, int gi, int gt, const double (&acc)[4][2]) {
#pragma unroll
  for (int t = 0; t < 4; ++t)
    *reinterpret_cast<double2*>(Ss + gi * WS_SLD + t * 8 + 2 * gt) = make_double2(acc[t][0], acc[t][1]);
}

// The product warp's part of one round: row blocks in pairs (b, b+1).  One pass
// over the H tile feeds both products — S_b over every row block and S_{b+1}
// over every block but b — so each B fragment is loaded once for two A
// fragments; S_{b+1} then gets block b's new rows (its "tail") once the row warp
// has solved block b.  The Gram fragments of the next pair are fetched while the
// row warp works (DMMA pipe idle).
template <int BT>
ENMF_DEV void bar_sync_n(int id) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(BT) : "memory"); }
template <int BT>
ENMF_DEV void bar_arrive_n(int id) { asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "n"(BT) : "memory"); }

// BT: threads on the hand-off barriers (64 = one product + one row warp; 128 = a team of
// three product warps and their row warp, sweep_t2)
template <int KS, int NB, int NT, int BT = 64>
ENMF_DEV void ws_producer_round(const double* Hs, double* Ss, const double2* gf, int gi, int gt, int bx0, int bx1,
                                int idS, int idH) {
  double A0[KS], A1[KS];
#pragma unroll
  for (int s = 0; s < KS; s += 2) {
    const double2 f0 = gf[(s / 2) * 32];
    const double2 f1 = gf[(KS / 2 + s / 2) * 32];
    A0[s] = f0.x; A0[s + 1] = f0.y;
    A1[s] = f1.x; A1[s + 1] = f1.y;
  }
#pragma unroll 1
  for (int b = 0; b < NB; b += 2) {
    if (b > 0) bar_sync_n<BT>(idH);                // rows of block b-1 are final in the tile
    double acc0[4][2], acc1[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) acc0[t][0] = acc0[t][1] = acc1[t][0] = acc1[t][1] = 0.0;
#pragma unroll
    for (int j = 0; j < KS / 2; ++j) {     // (block b's fragments of A1 are zero: see ws_prep)
      double2 p[4];
      ws_ldb<NT>(Hs, j, gt, bx0, bx1, p);
      ws_mma2<NT>(acc0, A0[2 * j], A0[2 * j + 1], p);
      ws_mma2<NT>(acc1, A1[2 * j], A1[2 * j + 1], p);
    }
    ws_store_s(Ss, gi, gt, acc0);
    bar_arrive_n<BT>(idS);                          // S_b ready: the row warp solves block b
    // while it does: this pair's tail fragments and the next pair's Gram fragments
    const double2 tl = gf[(16 * KS * KS + (b >> 1) * 64) / 2];   // Gf tails (ws_prep)
    if (b + 2 < NB) {
#pragma unroll
      for (int s = 0; s < KS; s += 2) {
        const double2 f0 = gf[(((b + 2) * KS / 2) + s / 2) * 32];
        const double2 f1 = gf[(((b + 3) * KS / 2) + s / 2) * 32];
        A0[s] = f0.x; A0[s + 1] = f0.y;
        A1[s] = f1.x; A1[s + 1] = f1.y;
      }
    }
    bar_sync_n<BT>(idH);                            // block b solved
    {
      double2 p[4];
      ws_ldb<NT>(Hs, b, gt, bx0, bx1, p);
      ws_mma2<NT>(acc1, tl.x, tl.y, p);
    }
    ws_store_s(Ss, gi, gt, acc1);
    bar_arrive_n<BT>(idS);                          // S_{b+1} ready
  }
}

// Persistent sweep kernels: grid-wide end of sweep `sw` — the stall rule on the total gain
// (nnls.hpp:172-173).  Single GPU: every CTA forms the same fixed-order total once all
// partials are in and decides itself; sharded: the last CTA exchanges the gain with the other
// ranks and publishes the decision.  Returns 1 to continue (same value in every thread).
// bid / nblk: this CTA's index and the CTA count of its grid (of its virtual rank's share of the
// grid in the virtual-rank sweep_tm).
ENMF_DEV int grid_decision(const Args& a, double gain, int nf, int sw, double& first_total, double* red,
                           unsigned bid = blockIdx.x, unsigned nblk = gridDim.x) {
  __shared__ int s_dec;
  const double bg = block_reduce_sum_any(__dadd_rn(gain, gain), red);   // gains are accumulated halved
  const int bnf = __syncthreads_or(nf);
  const unsigned target = (unsigned)(sw + 1) * nblk;
  // partials double-buffered by sweep parity: a CTA that has already decided sweep sw and
  // runs ahead writes its sweep sw+1 partial into the other half, never into the one a slower
  // CTA may still be summing (it can only come back to this half after every CTA has arrived
  // at sweep sw+1, i.e. after every CTA finished reading sweep sw's partials)
  double* part = a.part + (sw & 1) * nblk;
  int* part_nf = a.part_nf + (sw & 1) * nblk;
  if (threadIdx.x == 0) {
    part[bid] = bg;
    part_nf[bid] = bnf;
    __threadfence();
    const unsigned prev = atomicAdd(&a.ctl->arrive, 1u);
    s_dec = prev == target - 1 ? 1 : 0;      // this CTA arrived last (used when sharded)
  }
  if (!a.dv) {
    if (threadIdx.x == 0) {
      unsigned e;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(e) : "l"(&a.ctl->arrive) : "memory");
      } while (e < target);
    }
    __syncthreads();
    double v = 0.0;
    int f = 0;
    for (int b = threadIdx.x; b < (int)nblk; b += blockDim.x) {
      v = __dadd_rn(v, __ldcg(part + b));
      f |= __ldcg(part_nf + b);
    }
    const double total = block_reduce_sum_any(v, red);
    f = __syncthreads_or(f);
    if (sw == 0) first_total = total;
    const bool stop = (sw + 1 >= a.max_sweeps) ||
                      (total <= __dmul_rn(a.stall, first_total < 0.0 ? 0.0 : first_total));
    if (bid == 0 && threadIdx.x == 0) finish_sweep(a, total, f);   // bookkeeping (same rule)
    __syncthreads();
    return stop ? 0 : 1;
  }
  __syncthreads();
  if (s_dec) {
    __threadfence();
    double v = 0.0;
    int f = 0;
    for (int b = threadIdx.x; b < (int)nblk; b += blockDim.x) {
      v = __dadd_rn(v, __ldcg(part + b));
      f |= __ldcg(part_nf + b);
    }
    double total = block_reduce_sum_any(v, red);
    f = __syncthreads_or(f);
    if (threadIdx.x == 0) {
      dist::allreduce_gain(*a.dv, total, f, &total, &f);
      finish_sweep(a, total, f);
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(&a.ctl->epoch), "r"((unsigned)(sw + 1)) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned e;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(e) : "l"(&a.ctl->epoch) : "memory");
    } while (e < (unsigned)(sw + 1));
    s_dec = *(volatile int*)&a.ctl->cont;
  }
  __syncthreads();
  return s_dec;
}

// PERSIST: one launch runs every sweep of the solve.  Between sweeps the CTAs
// meet at a grid-wide decision point (the last CTA to arrive sums the per-CTA
// gains in fixed order, applies the stall rule — after the cross-GPU gain
// exchange when sharded — and publishes it through ctl->epoch), and the rounds
// alternate direction so the tile a pair finished a sweep with is the one it
// starts the next sweep with, already in shared memory.  Requires all CTAs to be
// co-resident (cooperative launch, one CTA per SM).
template <int RMAX, bool PERSIST = false>
__global__ void __launch_bounds__(256, 1) sweep_ws(Args a, long ntiles) {
  constexpr int NB = RMAX / 8;
  constexpr int KS = RMAX / 4;
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[256 + 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp & 3;
  const bool producer = warp < 4;
  double* Hs = sm + pair * (RMAX * 32);
  double* Ss = sm + 4 * RMAX * 32 + pair * 8 * WS_SLD;
  // per row block: lower triangle G[8b+l][8b+i] (i < l) at l(l-1)/2 + i, G_kk/2 at 28 + l,
  // 1/G_kk at 36 + l (padding rows: unit diagonal)
  double* Gc = sm + 4 * (RMAX * 32 + 8 * WS_SLD);
  const int r = a.r;
  for (int e = threadIdx.x; e < NB * 48; e += 256) {
    const int b = e / 48, j = e % 48;
    double v = 0.0;
    if (j < 28) {
      int l = 1;
      while (l * (l + 1) / 2 <= j) ++l;
      const int i = j - l * (l - 1) / 2, k = 8 * b + l, c = 8 * b + i;
      // scaled by the row's inverse diagonal: the row pass carries t = b / G_kk directly
      v = (k < r && c < r) ? __dmul_rn(a.G[(long)k * r + c], __ddiv_rn(1.0, a.G[(long)k * r + k])) : 0.0;
    } else if (j < 44) {
      const int k = 8 * b + ((j - 28) & 7);
      const double d = k < r ? a.G[(long)k * r + k] : 1.0;
      v = j < 36 ? __dmul_rn(0.5, d) : __ddiv_rn(1.0, d);
    }
    Gc[e] = v;
  }
  __syncthreads();

  const int idS = 1 + pair, idH = 5 + pair, idP = 9 + pair;
  const long P = (long)gridDim.x * 4, q = (long)blockIdx.x * 4 + pair;
  const long tq0 = q * ntiles / P, cnt = (q + 1) * ntiles / P - tq0;
  const int rounds = (int)((cnt + 3) / 4);
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  double gain = 0.0;
  int nf = 0;
  double first_total = 0.0;                 // persistent: the first sweep's total gain (stall rule)
  const int gi = lane >> 2, gt = lane & 3;
  // this lane's two 16-byte B-fragment chunks (tiles 0,1 and 2,3) within a row k with k & 3 == gt
  const int swz = ((gt & 1) << 2) | (gt >> 1);
  const int bx0 = 2 * ((2 * gi) ^ swz), bx1 = 2 * ((2 * gi + 1) ^ swz);
  const double2* gf = reinterpret_cast<const double2*>(a.Gf) + lane;
  int hoff[4];                              // swizzled position of column `lane` in a row k, by k & 3
#pragma unroll
  for (int j = 0; j < 4; ++j) hoff[j] = ws_pos(j, lane) - j * 32;

  for (int sw = 0;; ++sw) {
  for (int i = 0; i < rounds; ++i) {
    const int rd = (PERSIST && (sw & 1)) ? rounds - 1 - i : i;
    const long ta = tq0 + (long)rd * cnt / rounds;
    const int nt = (int)(tq0 + (long)(rd + 1) * cnt / rounds - ta);
    const long col0 = ta * 8;
    // stage this round's 32 columns of H (zero outside r × N and past nt tiles);
    // persistent: the first round of a later sweep is still in shared memory
    nb_sync(idP);                           // previous round done with the tiles
    if (!(PERSIST && sw > 0 && i == 0)) {
      const int c = lane;
      const long col = col0 + c;
      const bool okc = c < nt * 8 && col < a.N;
      const double* sp = src + col;
      for (int k = producer ? 0 : 1; k < RMAX; k += 2) {
        const bool ok = okc && k < r;
        const unsigned dst = (unsigned)__cvta_generic_to_shared(Hs + ws_pos(k, c));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst),
                     "l"(ok ? sp + (long)k * a.ld : src), "r"(ok ? 8 : 0));
      }
      asm volatile("cp.async.wait_all;\n" ::);
    }
    nb_sync(idP);

    if (producer) {
      switch (nt) {
        case 4: ws_producer_round<KS, NB, 4>(Hs, Ss, gf, gi, gt, bx0, bx1, idS, idH); break;
        case 3: ws_producer_round<KS, NB, 3>(Hs, Ss, gf, gi, gt, bx0, bx1, idS, idH); break;
        case 2: ws_producer_round<KS, NB, 2>(Hs, Ss, gf, gi, gt, bx0, bx1, idS, idH); break;
        default: ws_producer_round<KS, NB, 1>(Hs, Ss, gf, gi, gt, bx0, bx1, idS, idH); break;
      }
    } else {
      // predicated loads / stores with running row pointers (no branches, no per-row 64-bit
      // multiplies): invalid lanes read zeros and store nothing; rows past r are uniform
      const long col = col0 + lane;
      const bool valid = lane < nt * 8 && col < a.N;
      const long ld = a.ld, ld8 = 8 * ld;
      const double* cp = a.C + (valid ? col : 0);   // row 8b of this lane's column
      double* hp = a.H + (valid ? col : 0);
      double cn[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) cn[i] = (valid && i < r) ? cp[i * ld] : 0.0;
      int hmax = 0;                         // high words of the stored h (>= 0): +inf is 0x7FF00000
#pragma unroll 1
      for (int b = 0; b < NB; ++b) {
        double bb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) bb[i] = cn[i];
        if (b + 1 < NB) {
          const double* q = cp + ld8;
#pragma unroll
          for (int i = 0; i < 8; ++i) cn[i] = (valid && 8 * (b + 1) + i < r) ? q[i * ld] : 0.0;
        }
        // this block's lower triangle, half diagonal and inverse diagonal (broadcast loads)
        double gc[48];
        {
          const double2* gb = reinterpret_cast<const double2*>(Gc + b * 48);
#pragma unroll
          for (int j = 0; j < 22; ++j) {
            const double2 v = gb[j];
            gc[2 * j] = v.x;
            gc[2 * j + 1] = v.y;
          }
        }
        nb_sync(idS);
        double* hrow = Hs + 8 * b * 32;
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          // t = (C - S)/G_kk for all 8 rows up front; the chain then needs no multiply:
          // h_i = max(t_i, 0), t_l -= (G_li/G_ll) h_i
          bb[i] = __dmul_rn(__dsub_rn(bb[i], Ss[i * WS_SLD + lane]), gc[36 + i]);
          x[i] = hrow[i * 32 + hoff[i & 3]];
        }
        double hv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double h = pos_part_ws(bb[i]);
          hv[i] = h;
#pragma unroll
          for (int l = i + 1; l < 8; ++l) bb[l] = fma(-gc[l * (l - 1) / 2 + i], h, bb[l]);
          hrow[i * 32 + hoff[i & 3]] = h;
          // G_kk((x-t)² - (h-t)²) = (x-h)·(G_kk/2)·(x+h-2t)·2, accumulated halved
          const double u = __dsub_rn(x[i], h), v = __dadd_rn(x[i], h);
          gain = fma(__dmul_rn(u, gc[28 + i]), fma(-2.0, bb[i], v), gain);
        }
        if (b + 1 < NB) nb_arrive(idH);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (valid && 8 * b + i < r) hp[i * ld] = hv[i];
          hmax = max(hmax, __double2hiint(hv[i]));
        }
        cp += ld8;
        hp += ld8;
      }
      nf |= hmax >= 0x7FF00000;
    }
  }
  if (!PERSIST) break;
  // ---- grid-wide end of sweep `sw`: stall rule on the total gain ----
  {
    const int cont = grid_decision(a, gain, nf, sw, first_total, red);
    if (!cont) break;
    gain = 0.0;
    nf = 0;
    src = a.H;
  }
  }
  if (!PERSIST) {
    const double bg = block_reduce_sum_any(__dadd_rn(gain, gain), red);
    nf = __syncthreads_or(nf);
    last_block_reduce_n<256>(a, bg, nf, red);
  }
}

// ---- bitwise-faithful sweep (hals_row_update_impl order) -----------------
__global__ void __launch_bounds__(NT) sweep_exact(Args a) {
  if (sweep_skipped(a)) return;
  const int t = blockIdx.x * NT + threadIdx.x;
  if (t >= a.N) return;
  const int r = a.r;
  if (a.ctl->sweeps == 0) {
    for (int j = 0; j < r; ++j) a.H[(long)j * a.ld + t] = a.Hin[(long)j * a.ld + t];
  }
  for (int k = 0; k < r; ++k) {
    const double gkk = a.G[k * r + k];
    double b = a.C[(long)k * a.ld + t];
    for (int j = 0; j < r; ++j) {
      if (j == k) continue;
      const double gkj = a.G[k * r + j];
      if (gkj == 0.0) continue;
      b = __dsub_rn(b, __dmul_rn(gkj, a.H[(long)j * a.ld + t]));
    }
    const double hk = a.H[(long)k * a.ld + t];
    const double target = __ddiv_rn(b, gkk);
    const double next = target > 0.0 ? target : 0.0;
    const double d_old = __dsub_rn(hk, target);
    const double d_new = __dsub_rn(next, target);
    a.terms[(long)k * a.N + t] = __dsub_rn(__dmul_rn(d_old, d_old), __dmul_rn(d_new, d_new));
    a.H[(long)k * a.ld + t] = next;
  }
}

// gain = sum_k G[k][k] * (sum_t terms[k][t])  in the reference's order.
__global__ void __launch_bounds__(NT) gain_exact(Args a) {
  if ((a.st && !dev_active(a.st)) || !*(volatile int*)&a.ctl->cont) return;  // sweep_exact set cond
  __shared__ double rowgain[1024];
  const int r = a.r;
  for (int k = threadIdx.x; k < r; k += NT) {
    double gk = 0.0;
    const double* tk = a.terms + (long)k * a.N;
    for (int t = 0; t < a.N; ++t) gk = __dadd_rn(gk, tk[t]);
    rowgain[k < 1024 ? k : 1023] = __dmul_rn(a.G[k * r + k], gk);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double gain = 0.0;
    for (int k = 0; k < r; ++k) gain = __dadd_rn(gain, rowgain[k]);
    int nf = 0;
    for (int k = 0; k < r && !nf; ++k)
      for (int t = 0; t < a.N; ++t)
        if (!isfinite(a.H[(long)k * a.ld + t])) { nf = 1; break; }
    finish_sweep(a, gain, nf);
  }
}

// Resets the control block at the start of a solve.
__global__ void reset_ctl(HalsCtl* c, const DevState* st) {
  if (st && !dev_active(st)) return;
  c->first_gain = 0.0;
  c->last_gain = 0.0;
  c->sweeps = 0;
  c->cont = 1;
  c->nonfinite = 0;
  c->arrive = 0;
  c->epoch = 0;
}

}  // namespace hals

// hals_rl.cuh — HALS sweeps of the TF32 variant (ENMF_PRECISION_TF32, r <= 128) on the
// tcgen05 tensor cores: RIGHT-LOOKING blocked Gauss-Seidel with the residual in tensor memory
// (nnls.hpp:111-176; the variant's contract is the final relative error within 1e-4 of FP64).
//
// The left-looking sweeps (sweep_tm, sweep_tf32) form S_b = G[b rows, :]·H before every 8-row
// block: M = 8 per product, which only mma.sync shapes fit.  Here the residual
//     Rᵀ[column][k] = C[k][column] − Σ_j G[k][j]·H[j][column]
// of the CTA's ≤ 256 columns lives in TMEM for the whole inner solve (two accumulator tiles of
// 128 lanes × 128 FP32 columns: lane = column of H, TMEM column = row k), and is kept current
// by RANK-8 UPDATES on the tensor core: once the 8 rows of block b are solved,
//     Rᵀ += (−ΔH_bᵀ) · G[b rows, :]        one tcgen05.mma.kind::tf32, M = 128, N = 128, K = 8
// with A = the 128 columns' eight −Δh values, written by the row threads straight into eight
// TMEM columns (tcgen05.st → TS-form MMA, no shared-memory round trip), and B = block b's Gram
// rows from shared memory (K-major core-matrix tiles, staged once per solve).  The row pass of a
// block is one thread per column: r_k from its TMEM lane (tcgen05.ld.32x32b), t = h + r/G_kk,
// h' = max(t, 0), the in-block chain r_l −= G_lk·Δh_k in FP32, the gain term.  The errors of the
// TF32 products scale with Δh (they vanish as the solve converges) instead of with H as in the
// left-looking form; only the first residual R = C − G·H0 is a full TF32 product, formed with H0
// split into a TF32 head and tail (two MMAs per k-step) against TF32-rounded G.
//
// Per CTA: two independent column groups (warps 0-3 ↔ tile 0, warps 4-7 ↔ tile 1), each with its
// own mbarrier, named barrier and issuing thread, so one group's MMA round trip overlaps the
// other's row pass.  H itself (the iterate, FP32) sits in shared memory in the A-operand layout
// (used as the SS-form A of the first product, then as plain storage).  The kernel is resident
// only: the launcher uses it when every CTA's columns fit its two tiles (N <= 256·grid; and
// N >= 256, below which the per-solve staging outweighs it) and falls back to sweep_tf32
// otherwise.  Rows past r are padding (zero Gram rows, unit diagonal); only ⌈r/8⌉ blocks run.
// Stall decision: speculative on one GPU (a ninth warp decides sweep s while the compute warps run
// s+1, see the sweep loop); grid_decision (hals.cuh) when sharded.  Grid-wide stall decision: grid_decision (hals.cuh).
#pragma once

#include "hals.cuh"
#include "sweep_tf32.cuh"
#include "tc.cuh"

namespace hals {

constexpr int RL_GB = 16 * 4096;        // B tiles of G (TF32): 16 row blocks × (128 n × 8 k × 4 B)
constexpr int RL_HA = 128 * 128 * 4;    // one tile of Hᵀ in the K-major A layout (128 m × 128 k)
constexpr int RL_GC = 16 * 48 * 4;      // row-pass constants per block (FP32)
constexpr int rl_smem_bytes() { return 1024 + RL_GB + 2 * RL_HA + RL_GC + 64; }

// canonical no-swizzle K-major tiles (core matrix = 8 rows × 16 B):
// A (m = column of H, k = row): core matrices adjacent along K 128 B apart, 8-row groups 4 KB apart
ENMF_DEV int rl_a_off(int m, int k) { return (m >> 3) * 4096 + (k >> 2) * 128 + (m & 7) * 16 + (k & 3) * 4; }
// B of block b (n = row index of G, kk = row within the block): K halves 128 B apart, groups 256 B
ENMF_DEV int rl_b_off(int b, int n, int kk) { return b * 4096 + (n >> 3) * 256 + (kk >> 2) * 128 + (n & 7) * 16 + (kk & 3) * 4; }

ENMF_DEV void rl_ld8(uint32_t ta, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(ta));
}
ENMF_DEV void rl_wait_ld8(uint32_t (&v)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
               :
               : "memory");
}
ENMF_DEV void rl_st8(uint32_t ta, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
ENMF_DEV void rl_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
ENMF_DEV void rl_proxy_fence() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
ENMF_DEV void rl_bar(int id) { asm volatile("bar.sync %0, 128;\n" ::"r"(id) : "memory"); }

// D[tmem] += A[tmem: 128 lanes × 8 TF32 columns] · B[smem]ᵀ (TS form)
ENMF_DEV void rl_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc)
      : "memory");
}

template <int RMAX>
__global__ void __launch_bounds__(288, 1) sweep_rl(Args a) {
  static_assert(RMAX == 128, "two 128 × 128 residual tiles");
  constexpr int NB = RMAX / 8;
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(128) uint8_t rl_raw[];     // (no-swizzle operand tiles: 16-byte alignment suffices)
  uint8_t* sm = rl_raw;
  uint8_t* Gb = sm;                                        // B tiles
  uint8_t* Ha = sm + RL_GB;                                // [tile] Hᵀ, A layout
  float* Gc = reinterpret_cast<float*>(sm + RL_GB + 2 * RL_HA);   // [NB][48]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + RL_GB + 2 * RL_HA + RL_GC);   // one per tile group
  __shared__ double red[256 + 33];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool helper = warp == 8;                           // ninth warp: the stall decision (speculative path)
  const int tile = (warp >> 2) & 1, quarter = warp & 3;
  const int mloc = 32 * quarter + lane;                    // this thread's column within its tile
  const int r = a.r;
  const int nbr = (r + 7) >> 3;                            // row blocks in use (r <= 128)

  // ---- per-solve staging: Gram B tiles (TF32, round to nearest) and row-pass constants
#pragma unroll 1
  for (int e0 = threadIdx.x; e0 < NB * 128 * 8 && !helper; e0 += 256 * 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {                          // 8 loads in flight
      const int e = e0 + 256 * u, row = e >> 7, n = e & 127;
      v[u] = (row < r && n < r) ? (float)a.G[(long)row * r + n] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + 256 * u, row = e >> 7, n = e & 127;
      *reinterpret_cast<float*>(Gb + rl_b_off(row >> 3, n, row & 7)) = tf32_round(v[u]);
    }
  }
  for (int e = threadIdx.x; e < NB * 48 && !helper; e += 256) {
    const int b = e / 48, j = e % 48;
    double v = 0.0;
    if (j < 28) {
      int l = 1;
      while (l * (l + 1) / 2 <= j) ++l;
      const int i = j - l * (l - 1) / 2, k = 8 * b + l, c = 8 * b + i;
      v = (k < r && c < r) ? a.G[(long)k * r + c] : 0.0;
    } else if (j < 44) {
      const int k = 8 * b + ((j - 28) & 7);
      const double d = k < r ? a.G[(long)k * r + k] : 1.0;
      v = j < 36 ? 0.5 * d : 1.0 / d;
    }
    Gc[e] = (float)v;
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(mbar, 1);
    tc::mbar_init(mbar + 1, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
  rl_proxy_fence();                                        // B tiles: generic-proxy stores → tensor core reads
  tc::fence_before();
  __syncthreads();
  tc::fence_after();

  // this CTA's columns [c0, c0 + cnt), cnt <= 256; tile 0 = the first 128, tile 1 = the rest
  const long c0 = (long)blockIdx.x * a.N / gridDim.x, c1 = (long)(blockIdx.x + 1) * a.N / gridDim.x;
  const int cnt = (int)(c1 - c0);
  const int tcols = tile == 0 ? min(cnt, 128) : max(cnt - 128, 0);   // columns of this thread's tile
  const bool active = !helper && tcols > 0;                // (warp-uniform, group-uniform)
  const bool valid = mloc < tcols;
  const long col = c0 + tile * 128 + mloc;
  const uint32_t tR = tmem_base + (uint32_t)(tile * 128) + ((uint32_t)(32 * quarter) << 16);   // residual tile
  const uint32_t tS = tmem_base + 256u + (uint32_t)(tile * 8) + ((uint32_t)(32 * quarter) << 16);   // −Δ staging
  const uint32_t dR = tmem_base + (uint32_t)(tile * 128), dS = tmem_base + 256u + (uint32_t)(tile * 8);
  uint8_t* Ht = Ha + tile * RL_HA;
  uint64_t* mb = mbar + tile;
  uint32_t mph = 0;                                        // mbarrier phase of this group
  constexpr uint32_t IDESC = tc::idesc_tf32(128, 128);
  const uint64_t dB0 = tc::desc_noswz(tc::smem_u32(Gb), 128, 256);
  const uint64_t dA0 = tc::desc_noswz(tc::smem_u32(Ht), 128, 4096);
  const bool issuer = !helper && (threadIdx.x & 127) == 0;
  const int bar_id = 1 + tile;
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  const double* hsrc = src + (valid ? col : 0);
  const double* csrc = a.C + (valid ? col : 0);

  if (active) {
    // ---- R = C − G·H0: C into the residual tile, then two SS-form passes over k with A = −head(H0)
    // and A = −tail(H0) (TF32 head/tail split of the FP32 value)
#pragma unroll 2
    for (int k0 = 0; k0 < RMAX; k0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[i] = __float_as_uint((valid && k0 + i < r) ? (float)csrc[(long)(k0 + i) * a.ld] : 0.f);
      rl_st8(tR + k0, v);
    }
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {               // pass 2 leaves the iterate itself (FP32, unrounded)
#pragma unroll 1
      for (int k0 = 0; k0 < RMAX; k0 += 16) {
        float h[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) h[i] = (valid && k0 + i < r) ? (float)hsrc[(long)(k0 + i) * a.ld] : 0.f;
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          float o[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float hi = tf32_round(h[i + u]);
            o[u] = pass == 0 ? -hi : pass == 1 ? -tf32_round(h[i + u] - hi) : h[i + u];
          }
          *reinterpret_cast<float4*>(Ht + rl_a_off(mloc, k0 + i)) = make_float4(o[0], o[1], o[2], o[3]);
        }
      }
      if (pass == 2) break;
      rl_wait_st();
      rl_proxy_fence();
      tc::fence_before();
      rl_bar(bar_id);
      if (issuer) {
        tc::fence_after();
#pragma unroll 1
        for (int s = 0; s < nbr; ++s)
          tc::mma_tf32(dR, dA0 + (uint64_t)((s * 256) >> 4), dB0 + (uint64_t)((s * 4096) >> 4), IDESC, 1u);
        tc::commit(mb);
      }
      tc::mbar_wait(mb, mph);
      mph ^= 1;
      tc::fence_after();
    }
    __syncwarp();
  }

  // Speculative stall decision (single GPU, as in sweep_tm): the grid-wide decision costs 3.2 µs
  // per sweep when every CTA waits for it (profiles/r02_sweep_rl_scan.txt), so sweep s only hands
  // its gain partial to the CTA's ninth warp and the eight compute warps go on with sweep s+1.
  // The ninth warp publishes the partial, waits for every CTA's, forms the fixed-order total and
  // posts a "stop" in shared memory, which each column group picks up at its next step barrier
  // (and everybody at the end of the next sweep, before which sweep s must be decided).  A "stop" on s discards s+1: every block's old rows are saved before they are
  // overwritten — blocks 0..14 in the 240 TMEM columns left over, block 15 in registers — so the
  // blocks already redone are restored and the others still hold sweep s.  Sharded solves keep the
  // synchronous grid_decision (its cross-GPU exchange).
  const bool spec = a.dv == nullptr;
  const uint32_t tN = tmem_base + 272u + (uint32_t)(tile * 120) + ((uint32_t)(32 * quarter) << 16);   // saved rows of blocks 0..14
  __shared__ float s_wg[2][8];
  __shared__ int s_wnf[2][8];
  __shared__ int s_stop_at;                 // sweep decided to be the last (-1: none yet)
  __shared__ int s_decided;                 // last sweep whose decision is in
  __shared__ int g_stop[2][2];              // [column group][step parity]: the group's uniform view of "stop"
  if (threadIdx.x == 0) {
    s_stop_at = -1;
    s_decided = -1;
  }
  __syncthreads();
  int restore_upto = 0;                     // blocks [0, restore_upto) come back from the saved rows
  float xlast[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  double first_total = 0.0;
  auto arrived = [&]() {
    unsigned e;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(e) : "l"(&a.ctl->arrive) : "memory");
    return e;
  };
  // (ninth warp) decision on sweep s once every CTA has published it; CTA 0 does the bookkeeping
  auto decide = [&](int s) {
    while (arrived() < (unsigned)(s + 1) * gridDim.x) __nanosleep(100);
    const double* part = a.part + (s & 1) * gridDim.x;
    const int* part_nf = a.part_nf + (s & 1) * gridDim.x;
    double v = 0.0;
    int f = 0;
    for (int bb = lane; bb < (int)gridDim.x; bb += 32) {
      v = __dadd_rn(v, __ldcg(part + bb));
      f |= __ldcg(part_nf + bb);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    f = __any_sync(0xffffffffu, f) ? 1 : 0;
    if (s == 0) first_total = v;
    const bool stop = (s + 1 >= a.max_sweeps) || (v <= __dmul_rn(a.stall, first_total < 0.0 ? 0.0 : first_total));
    if (blockIdx.x == 0 && lane == 0) finish_sweep(a, v, f);
    if (lane == 0) {
      if (stop) *(volatile int*)&s_stop_at = s;
      __threadfence_block();
      *(volatile int*)&s_decided = s;
    }
  };
  for (int sw = 0;; ++sw) {
    float gain = 0.f;
    int hmax = 0;
    bool stopped = false;
    if (active) {
#pragma unroll 1
      for (int b = 0; b < nbr; ++b) {
        // everything that does not need the residual first: constants and the block's old rows
        float gc[44];
#pragma unroll
        for (int j = 0; j < 11; ++j) {
          const float4 v = reinterpret_cast<const float4*>(Gc + b * 48)[j];
          gc[4 * j] = v.x; gc[4 * j + 1] = v.y; gc[4 * j + 2] = v.z; gc[4 * j + 3] = v.w;
        }
        const float4 h0 = *reinterpret_cast<const float4*>(Ht + rl_a_off(mloc, 8 * b));
        const float4 h1 = *reinterpret_cast<const float4*>(Ht + rl_a_off(mloc, 8 * b + 4));
        float x[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        if (sw > 0 || b > 0) {                             // the previous block's update is in
          tc::mbar_wait(mb, mph);
          mph ^= 1;
          tc::fence_after();
        }
        uint32_t rv[8];
        rl_ld8(tR + 8 * b, rv);
        rl_wait_ld8(rv);
        float rr[8], hn[8];
        uint32_t dv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) rr[k] = __uint_as_float(rv[k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float t = fmaf(rr[k], gc[36 + k], x[k]);   // h + r/G_kk
          const float h = fmaxf(t, 0.f);                   // NaN -> 0, as `t > 0 ? t : 0`
          const float d = h - x[k];
          hn[k] = h;
#pragma unroll
          for (int l = k + 1; l < 8; ++l) rr[l] = fmaf(-gc[l * (l - 1) / 2 + k], d, rr[l]);
          dv[k] = __float_as_uint(tf32_round(-d));
          // G_kk((x−t)² − (h−t)²) = (x−h)(x+h−2t)·G_kk, accumulated halved
          gain = fmaf(-d * gc[28 + k], fmaf(-2.f, t, x[k] + h), gain);
          hmax = max(hmax, __float_as_int(h));
        }
        rl_st8(tS, dv);
        if (spec) {                                        // the rows this step overwrites
          if (b < 15) {
#pragma unroll
            for (int k = 0; k < 8; ++k) rv[k] = __float_as_uint(x[k]);
            rl_st8(tN + 8 * b, rv);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) xlast[k] = x[k];
          }
        }
        *reinterpret_cast<float4*>(Ht + rl_a_off(mloc, 8 * b)) = make_float4(hn[0], hn[1], hn[2], hn[3]);
        *reinterpret_cast<float4*>(Ht + rl_a_off(mloc, 8 * b + 4)) = make_float4(hn[4], hn[5], hn[6], hn[7]);
        rl_wait_st();
        tc::fence_before();
        if (spec && issuer && sw > 0) g_stop[tile][b & 1] = *(volatile int*)&s_stop_at == sw - 1;
        rl_bar(bar_id);
        if (issuer) {
          tc::fence_after();
          rl_mma_ts(dR, dS, dB0 + (uint64_t)((b * 4096) >> 4), IDESC);
          tc::commit(mb);
        }
        if (spec && sw > 0 && *(volatile int*)&g_stop[tile][b & 1]) {   // sweep sw is discarded
          restore_upto = b + 1;
          stopped = true;
          break;
        }
      }
    }
    const int nf = hmax >= 0x7F800000 ? 1 : 0;
    if (!spec) {
      const int cont = grid_decision(a, (double)gain, nf, sw, first_total, red);
      if (!cont) break;
      continue;
    }
    // ---- speculative end of sweep `sw`: the compute warps hand their gain partials to the ninth
    // warp without waiting for anybody (they only ARRIVE at the barrier it syncs on, ids 3 / 4 by
    // sweep parity), so the two column groups drift independently; they go on once sweep sw-1 is
    // decided, which it normally has been for most of a sweep
    const bool last = sw + 1 >= a.max_sweeps;              // the cap: no speculation past it
    if (!helper) {
      float g = gain + gain;                               // gains are accumulated halved
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) g += __shfl_xor_sync(0xffffffffu, g, off);
      const int f = __any_sync(0xffffffffu, nf) ? 1 : 0;
      if (lane == 0) {
        s_wg[sw & 1][warp] = g;
        s_wnf[sw & 1][warp] = f;
      }
      __syncwarp();
      asm volatile("bar.arrive %0, 288;\n" ::"r"(3 + (sw & 1)) : "memory");
      if (sw > 0) {
        while (*(volatile int*)&s_decided < sw - 1) {
        }
        if (*(volatile int*)&s_stop_at == sw - 1) {        // sweep sw-1 was the last: sweep sw is discarded
          if (!stopped) restore_upto = active ? nbr : 0;
          break;
        }
      }
      if (last) break;
    } else {
      asm volatile("bar.sync %0, 288;\n" ::"r"(3 + (sw & 1)) : "memory");
      if (sw > 0 && *(volatile int*)&s_stop_at == sw - 1) break;
      if (lane == 0) {                                     // this CTA's sweep-sw partial (fixed order over the warps)
        double g = 0.0;
        int f = 0;
        for (int w = 0; w < 8; ++w) {
          g = __dadd_rn(g, (double)s_wg[sw & 1][w]);
          f |= s_wnf[sw & 1][w];
        }
        a.part[(sw & 1) * gridDim.x + blockIdx.x] = g;
        a.part_nf[(sw & 1) * gridDim.x + blockIdx.x] = f;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(&a.ctl->arrive) : "memory");
      }
      __syncwarp();
      if (!last || blockIdx.x == 0) decide(sw);            // (at the cap: CTA 0 only, for the bookkeeping)
      if (last) break;
    }
  }
  // a discarded speculative sweep: the blocks it had already redone come back from the saved rows
  if (active && restore_upto > 0) {
#pragma unroll 1
    for (int b = 0; b < restore_upto; ++b) {
      float o[8];
      if (b < 15) {
        uint32_t rv[8];
        rl_ld8(tN + 8 * b, rv);
        rl_wait_ld8(rv);
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = __uint_as_float(rv[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = xlast[k];
      }
      *reinterpret_cast<float4*>(Ht + rl_a_off(mloc, 8 * b)) = make_float4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<float4*>(Ht + rl_a_off(mloc, 8 * b + 4)) = make_float4(o[4], o[5], o[6], o[7]);
    }
  }
  // the result: this CTA's columns of H (rows < r)
  if (active && valid)
    for (int k = 0; k < r; ++k) a.H[(long)k * a.ld + col] = (double)*reinterpret_cast<const float*>(Ht + rl_a_off(mloc, k));
  if (active) {                                            // drain the last MMA before the TMEM is freed
    tc::mbar_wait(mb, mph);
    tc::fence_after();
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace hals

// sweep_tf32.cuh — HALS sweeps of the TF32 variant (ENMF_PRECISION_TF32) on sm_100a.
//
// Same structure as hals::sweep_ws (persistent, one warp pair per SM sub-partition over 32
// columns, product warp / row warp alternating with named-barrier hand-offs, grid-wide stall
// decision), with the block products on the TF32 tensor cores: one
// mma.sync.m16n8k8.tf32 covers a PAIR of 8-row Gauss-Seidel blocks (rows 0-7 = block b,
// rows 8-15 = block b+1) for one 8-column tile — 8× the FP64 DMMA rate
// (profiles/r01_tf32_mma.txt).  Block b+1's rows see block b's columns only through a
// one-k-step "tail" MMA issued after the row warp has solved block b.  The H tile lives in
// shared memory in FP32, rounded to TF32 (round to nearest: the tensor cores would drop the
// low mantissa bits, a bias), the row pass runs in FP32, the gain is reduced in FP64.
// The variant's accuracy contract is the final relative error within 1e-4 of FP64.
#pragma once

#include "hals.cuh"

namespace hals {

constexpr int TF_SP = 40;   // S tile row stride (floats): conflict-free 8-byte fragment stores

template <int RMAX>
constexpr int tf_smem_bytes() {
  return (4 * (RMAX * 32 + 16 * TF_SP) + (RMAX / 8) * 48) * 4;
}

ENMF_DEV float tf32_round(float x) {
  unsigned t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(x));
  return __uint_as_float(t);
}

// position of (row k, column c) in the FP32 tile: 16-byte chunk (k, c & 7) holds the 4
// tiles' values of n-index c & 7, XOR-swizzled by the row so B-fragment loads are conflict-free
ENMF_DEV int tf_pos(int k, int c) { return k * 32 + (((c & 7) ^ (2 * (k & 3))) << 2) + (c >> 3); }

ENMF_DEV float pos_part_f(float t) {
  const int b = __float_as_int(t);
  return (b > 0 && b <= 0x7F800000) ? t : 0.0f;
}

// A fragments of m16n8k8.tf32 (row-major 16×8): for pair-block P (rows 16P..16P+15 = blocks
// 2P, 2P+1) and k-step j (columns 8j..8j+7): a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4],
// a3 = A[g+8][t+4], g = lane/4, t = lane%4.  Zero outside r×r, on/below the diagonal inside
// diagonal blocks, and for the block-(2P+1) rows in block 2P's columns (those enter through
// the tail, stored after the main fragments: rows 0-7 zero, rows 8-15 = G[2P+1 rows][2P cols]).
template <int RMAX>
__global__ void tf_prep(const double* G, int r, float4* Gf, const DevState* st, const HalsCtl* ctl) {
  if ((st && !dev_active(st)) || !ctl->cont) return;
  constexpr int NP = RMAX / 16, KJ = RMAX / 8;
  const int total = (NP * KJ + NP) * 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int lane = i & 31, w = i >> 5;
    const bool tail = w >= NP * KJ;
    const int P = tail ? w - NP * KJ : w / KJ, j = tail ? 2 * P : w % KJ;
    const int g = lane >> 2, t = lane & 3;
    float v[4];
    for (int e = 0; e < 4; ++e) {
      const int lr = g + ((e & 1) ? 8 : 0), lc = t + ((e & 2) ? 4 : 0);
      const int row = 16 * P + lr, col = 8 * j + lc;
      const int rb = row >> 3, cb = col >> 3;   // row / column blocks
      double x = 0.0;
      if (row < r && col < r) x = G[(long)row * r + col];
      if (rb == cb && (col & 7) <= (row & 7)) x = 0.0;   // diagonal block: strictly upper part
      if (!tail && (rb & 1) && cb == rb - 1) x = 0.0;     // block 2P+1 × block 2P: via the tail
      if (tail && !(lr >= 8)) x = 0.0;                   // tail: rows of block 2P+1 only
      v[e] = tf32_round((float)(-x));                     // negated: accumulate onto C
    }
    Gf[i] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

ENMF_DEV void tf_mma(float (&d)[4], const float4& a, float b0, float b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(__float_as_uint(a.x)), "r"(__float_as_uint(a.y)), "r"(__float_as_uint(a.z)),
                 "r"(__float_as_uint(a.w)), "r"(__float_as_uint(b0)), "r"(__float_as_uint(b1)));
}

// D fragments (rows g / g+8 = block b / b+1, columns 2t, 2t+1 of each tile) into the S tile
ENMF_DEV void tf_store_s(float* Ss, int g, int t, const float (&acc)[4][4], bool upper) {
#pragma unroll
  for (int tt = 0; tt < 4; ++tt) {
    const int col = tt * 8 + 2 * t;
    if (!upper) *reinterpret_cast<float2*>(Ss + g * TF_SP + col) = make_float2(acc[tt][0], acc[tt][1]);
    else *reinterpret_cast<float2*>(Ss + (g + 8) * TF_SP + col) = make_float2(acc[tt][2], acc[tt][3]);
  }
}

template <int RMAX>
ENMF_DEV void tf_producer_round(const Args& a, long col0, int nt, const float* Hs, float* Ss, const float4* gf,
                                int g, int t, int idS, int idH) {
  constexpr int NP = RMAX / 16, KJ = RMAX / 8;
  const int r = a.r;
  float4 A[KJ];
#pragma unroll
  for (int j = 0; j < KJ; ++j) A[j] = gf[j * 32];
#pragma unroll 1
  for (int P = 0; P < NP; ++P) {
    if (P > 0) nb_sync(idH);                 // block 2P-1 solved
    // accumulators start from C (the products are negated): rows 16P+g and 16P+8+g
    float acc[4][4];
#pragma unroll
    for (int tt = 0; tt < 4; ++tt) {
      const long c0 = col0 + tt * 8 + 2 * t;
      const int r0 = 16 * P + g, r1 = r0 + 8;
      const bool okt = tt < nt;
      const double* p0 = a.C + (long)r0 * a.ld + c0;
      const double* p1 = a.C + (long)r1 * a.ld + c0;
      acc[tt][0] = (okt && r0 < r && c0 < a.N) ? (float)p0[0] : 0.f;
      acc[tt][1] = (okt && r0 < r && c0 + 1 < a.N) ? (float)p0[1] : 0.f;
      acc[tt][2] = (okt && r1 < r && c0 < a.N) ? (float)p1[0] : 0.f;
      acc[tt][3] = (okt && r1 < r && c0 + 1 < a.N) ? (float)p1[1] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
      const float4 b0 = *reinterpret_cast<const float4*>(Hs + tf_pos(8 * j + t, g) - (g >> 3));
      const float4 b1 = *reinterpret_cast<const float4*>(Hs + tf_pos(8 * j + t + 4, g) - (g >> 3));
      tf_mma(acc[0], A[j], b0.x, b1.x);
      tf_mma(acc[1], A[j], b0.y, b1.y);
      tf_mma(acc[2], A[j], b0.z, b1.z);
      tf_mma(acc[3], A[j], b0.w, b1.w);
    }
    tf_store_s(Ss, g, t, acc, false);
    nb_arrive(idS);                          // C - S of block 2P
    const float4 tl = gf[(NP * KJ + P) * 32];
    if (P + 1 < NP) {
#pragma unroll
      for (int j = 0; j < KJ; ++j) A[j] = gf[((P + 1) * KJ + j) * 32];
    }
    nb_sync(idH);                            // block 2P solved
    {
      const int j = 2 * P;
      const float4 b0 = *reinterpret_cast<const float4*>(Hs + tf_pos(8 * j + t, g) - (g >> 3));
      const float4 b1 = *reinterpret_cast<const float4*>(Hs + tf_pos(8 * j + t + 4, g) - (g >> 3));
      tf_mma(acc[0], tl, b0.x, b1.x);
      tf_mma(acc[1], tl, b0.y, b1.y);
      tf_mma(acc[2], tl, b0.z, b1.z);
      tf_mma(acc[3], tl, b0.w, b1.w);
    }
    tf_store_s(Ss, g, t, acc, true);
    nb_arrive(idS);                          // C - S of block 2P+1
  }
}

template <int RMAX>
__global__ void __launch_bounds__(256, 1) sweep_tf32(Args a, long ntiles) {
  constexpr int NB = RMAX / 8;
  if (sweep_skipped(a)) return;
  extern __shared__ __align__(16) float smf[];
  __shared__ double red[256 + 33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp & 3;
  const bool producer = warp < 4;
  float* Hs = smf + pair * (RMAX * 32);
  float* Ss = smf + 4 * RMAX * 32 + pair * 16 * TF_SP;
  float* Gc = smf + 4 * (RMAX * 32 + 16 * TF_SP);   // per block: lower triangle, G_kk/2, 1/G_kk
  const int r = a.r;
  for (int e = threadIdx.x; e < NB * 48; e += 256) {
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
  __syncthreads();

  const int idS = 1 + pair, idH = 5 + pair, idP = 9 + pair;
  const long P = (long)gridDim.x * 4, q = (long)blockIdx.x * 4 + pair;
  const long tq0 = q * ntiles / P, cnt = (q + 1) * ntiles / P - tq0;
  const int rounds = (int)((cnt + 3) / 4);
  const double* src = (a.ctl->sweeps == 0) ? a.Hin : a.H;
  float gain = 0.f;
  double gain_d = 0.0;                      // per-round flush of the FP32 partial
  int nf = 0;
  double first_total = 0.0;
  const int g = lane >> 2, t = lane & 3;
  const float4* gf = reinterpret_cast<const float4*>(a.Gf) + lane;

  for (int sw = 0;; ++sw) {
    for (int i = 0; i < rounds; ++i) {
      const int rd = (sw & 1) ? rounds - 1 - i : i;
      const long ta = tq0 + (long)rd * cnt / rounds;
      const int nt = (int)(tq0 + (long)(rd + 1) * cnt / rounds - ta);
      const long col0 = ta * 8;
      nb_sync(idP);
      if (!(sw > 0 && i == 0)) {            // the first round of a later sweep is resident
        const int c = lane;
        const long col = col0 + c;
        const bool okc = c < nt * 8 && col < a.N;
        const double* sp = src + col;
        for (int k = producer ? 0 : 1; k < RMAX; k += 2)
          Hs[tf_pos(k, c)] = (okc && k < r) ? tf32_round((float)sp[(long)k * a.ld]) : 0.f;
      }
      nb_sync(idP);
      if (producer) {
        tf_producer_round<RMAX>(a, col0, nt, Hs, Ss, gf, g, t, idS, idH);
      } else {
        // predicated stores with a running row pointer (no branches, no per-row 64-bit multiplies)
        const long col = col0 + lane;
        const bool valid = lane < nt * 8 && col < a.N;
        const long ld = a.ld, ld8 = 8 * ld;
        double* hp = a.H + (valid ? col : 0);     // row 8b of this lane's column
        int hmax = 0;
#pragma unroll 1
        for (int b = 0; b < NB; ++b) {
          float gc[44];
#pragma unroll
          for (int j = 0; j < 11; ++j) {
            const float4 v = reinterpret_cast<const float4*>(Gc + b * 48)[j];
            gc[4 * j] = v.x; gc[4 * j + 1] = v.y; gc[4 * j + 2] = v.z; gc[4 * j + 3] = v.w;
          }
          nb_sync(idS);
          const float* srow = Ss + (b & 1) * 8 * TF_SP + lane;
          float bb[8], x[8], hv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            bb[k] = srow[k * TF_SP];
            x[k] = Hs[tf_pos(8 * b + k, lane)];
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float tv = bb[k] * gc[36 + k];
            const float h = pos_part_f(tv);
            hv[k] = h;
#pragma unroll
            for (int l = k + 1; l < 8; ++l) bb[l] = fmaf(-gc[l * (l - 1) / 2 + k], h, bb[l]);
            Hs[tf_pos(8 * b + k, lane)] = tf32_round(h);
            const float u = x[k] - h, v = x[k] + h;
            gain = fmaf(u, fmaf(gc[28 + k], v, -bb[k]), gain);
          }
          if (b + 1 < NB) nb_arrive(idH);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (valid && 8 * b + k < r) hp[k * ld] = (double)hv[k];
            hmax = max(hmax, __float_as_int(hv[k]));
          }
          hp += ld8;
        }
        nf |= hmax >= 0x7F800000;
        gain_d += (double)gain;
        gain = 0.f;
      }
    }
    const int cont = grid_decision(a, gain_d, nf, sw, first_total, red);
    if (!cont) break;
    gain_d = 0.0;
    nf = 0;
    src = a.H;
  }
}

}  // namespace hals

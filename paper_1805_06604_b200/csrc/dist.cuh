// dist.cuh — multi-GPU sharding of the hot path over NVLink/NVSwitch peer memory.
//
// rank p of P owns X[:, J_p] (column block, for W_yᵀX) and
// X[I_p, :] (row block, for X·Tᵀ) plus the matching shards H[:, J_p] and
// W[I_p, :].  Per outer iteration the only exchanges are
//   * all-gathers of the factor shards W_yᵀ[:, I_p] and T[:, J_p] into full
//     r×m / r×n replicas (every rank stores its shard straight into every
//     peer's replica through CUDA-IPC mapped peer pointers, then a barrier);
//   * sum-all-reduces of the r×r Gram partials and the error partials;
//   * one scalar sum (+ NaN flag) per HALS sweep for the global stall rule;
// all done by our own kernels with peer stores and epoch flags — no host
// round trip, everything stays inside the per-iteration CUDA graph.
// Reductions add the P contributions in rank order on every rank, so every
// rank holds bitwise-identical reduced values and takes identical decisions.
//
// Buffer layout of each rank's IPC allocation (DistShared):
//   flags[MAXP]            epoch written by peer q after its payload for that epoch
//   slots[2][MAXP][SLOT]   payloads, double-buffered by epoch parity
// A rank may only write epoch e+2 after every rank signalled e+1, i.e. after
// every rank finished reading epoch e, so two parities suffice.
#pragma once

#include "common.cuh"

namespace dist {

constexpr int MAXP = 8;

struct View {
  int rank, world;
  unsigned long long* flags[MAXP];   // flags array of rank q's shared block
  double* slots[MAXP];               // slots of rank q: [2][MAXP][slot]
  int slot;                          // doubles per (parity, sender) slot
  double* full_peer_w[MAXP];         // rank q's W_yᵀ replica (r×m)
  double* full_peer_t[MAXP];         // rank q's T replica (r×n)
  unsigned long long* epoch;         // device counter (this rank), identical sequence on all ranks
  int* error;                        // set on peer timeout
};

ENMF_DEV void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
ENMF_DEV unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Thread 0 of the calling block: publish `e` to every rank, then wait until
// every rank published `e` to us.  Times out after ~20 s (error flag).
ENMF_DEV void signal_and_wait(const View& v, unsigned long long e) {
  __threadfence_system();
  for (int q = 0; q < v.world; ++q) st_release_sys(v.flags[q] + v.rank, e);
  const unsigned long long t0 = globaltimer_ns();
  for (int q = 0; q < v.world; ++q) {
    while (ld_acquire_sys(v.flags[v.rank] + q) < e) {
      __nanosleep(64);
      if (globaltimer_ns() - t0 > 20000000000ULL) {
        atomicExch(v.error, 1);
        return;
      }
    }
  }
}

// Block-level sum-all-reduce of `count` doubles (count <= slot): every rank
// ends with out[i] = sum_q in[q][i], q ascending.  All threads participate.
ENMF_DEV void allreduce_block(const View& v, const double* in, int count, double* out) {
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) s_epoch = ++(*v.epoch);
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int par = (int)(e & 1ULL);
  for (int q = 0; q < v.world; ++q) {
    double* dst = v.slots[q] + ((long)par * MAXP + v.rank) * v.slot;
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = in[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) signal_and_wait(v, e);
  __syncthreads();
  const double* own = v.slots[v.rank] + (long)par * MAXP * v.slot;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double s = own[i];
    for (int q = 1; q < v.world; ++q) s = __dadd_rn(s, own[(long)q * v.slot + i]);
    out[i] = s;
  }
  __syncthreads();
}

// Single-thread max over ranks (BPP feasibility tolerance: max|C| of the whole cross product).
ENMF_DEV double allmax_scalar(const View& v, double x) {
  const unsigned long long e = ++(*v.epoch);
  const int par = (int)(e & 1ULL);
  for (int q = 0; q < v.world; ++q) v.slots[q][((long)par * MAXP + v.rank) * v.slot] = x;
  signal_and_wait(v, e);
  const double* own = v.slots[v.rank] + (long)par * MAXP * v.slot;
  double m = own[0];
  for (int q = 1; q < v.world; ++q) m = fmax(m, own[(long)q * v.slot]);
  return m;
}

// Single-thread scalar variant (the HALS sweep's last block): sums (gain, nf).
ENMF_DEV void allreduce_gain(const View& v, double gain, int nf, double* gsum, int* nfor) {
  const unsigned long long e = ++(*v.epoch);
  const int par = (int)(e & 1ULL);
  for (int q = 0; q < v.world; ++q) {
    double* dst = v.slots[q] + ((long)par * MAXP + v.rank) * v.slot;
    dst[0] = gain;
    dst[1] = (double)nf;
  }
  signal_and_wait(v, e);
  const double* own = v.slots[v.rank] + (long)par * MAXP * v.slot;
  double s = own[0];
  int f = own[1] != 0.0;
  for (int q = 1; q < v.world; ++q) {
    s = __dadd_rn(s, own[(long)q * v.slot]);
    f |= own[(long)q * v.slot + 1] != 0.0;
  }
  *gsum = s;
  *nfor = f;
}

// Barrier only (after the all-gather stores): thread 0 of the calling block.
ENMF_DEV void barrier_body(const View& v) {
  if (threadIdx.x == 0) {
    const unsigned long long e = ++(*v.epoch);
    signal_and_wait(v, e);
  }
}

// All-gather of a factor shard: local (r × cnt, row-major, ld cnt) is stored
// into columns [off, off+cnt) of every rank's replica (r × full, ld full).
// tid / nthreads: the calling thread's index among the threads that share the copy.
ENMF_DEV void scatter_body(const View& v, const double* __restrict__ local, int r, long cnt, long off, long full,
                           int which, long tid, long nthreads) {
  const long total = (long)r * cnt;
  for (int q = 0; q < v.world; ++q) {
    double* dst = which == 0 ? v.full_peer_w[q] : v.full_peer_t[q];
    for (long e = tid; e < total; e += nthreads) {
      const long k = e / cnt, j = e % cnt;
      dst[k * full + off + j] = local[e];
    }
  }
}

// Sum-all-reduce of a device array (count doubles) in place, one block.
__global__ void allreduce_inplace(const View* v, double* buf, int count, const DevState* st) {
  if (st && !dev_active(st)) return;
  allreduce_block(*v, buf, count, buf);
}

__global__ void barrier_k(const View* v, const DevState* st) {
  if (st && !dev_active(st)) return;
  barrier_body(*v);
}

__global__ void scatter_shard_k(const View* v, const double* __restrict__ local, int r, long cnt, long off, long full,
                                int which, const DevState* st) {
  if (st && !dev_active(st)) return;
  scatter_body(*v, local, r, cnt, off, full, which, blockIdx.x * (long)blockDim.x + threadIdx.x,
               (long)gridDim.x * blockDim.x);
}

// Self-test of the exchange primitives with `world` ranks on ONE GPU: block p of a cooperative
// launch (all blocks co-resident, so the spin-waits always make progress) plays rank p with its
// own View — own flags, slots, replicas and epoch counter, all in this process's memory — and
// runs `epochs` rounds of every exchange the engine uses: the block all-reduce (Gram / error
// partials), the scalar gain and max exchanges of the sweeps and BPP, and the shard all-gather +
// barrier.  out[p] receives what rank p ended up with, for the host to compare with the
// rank-ordered sums and across ranks (enmf_gpu_dist_selftest).
//   in:  [world][count]      per-rank contribution (round e uses in·(e+1))
//   red: [world][epochs][count] all-reduced values;  sc: [world][epochs][3] gain sum, flag, max
//   rep: each rank's r × full replica ends up holding round (epochs-1)'s shards of every rank
__global__ void selftest(const View* views, int count, int epochs, const double* in, double* red, double* sc,
                         double* stage, int r, long full) {
  const View& v = views[blockIdx.x];
  const int p = v.rank, P = v.world;
  double* mine = stage + (long)p * (count + (long)r * full);     // [count] contribution | [r × cnt] shard
  double* shard = mine + count;
  const long base = full / P, extra = full % P;
  const long cnt = base + (p < extra ? 1 : 0), off = p * base + (p < extra ? p : extra);
  for (int e = 0; e < epochs; ++e) {
    for (int i = threadIdx.x; i < count; i += blockDim.x) mine[i] = __dmul_rn(in[(long)p * count + i], (double)(e + 1));
    __syncthreads();
    allreduce_block(v, mine, count, red + ((long)p * epochs + e) * count);
    if (threadIdx.x == 0) {
      double g;
      int f;
      allreduce_gain(v, __dmul_rn(in[(long)p * count], (double)(e + 2)), (p == e % P) ? 1 : 0, &g, &f);
      double* o = sc + ((long)p * epochs + e) * 3;
      o[0] = g;
      o[1] = (double)f;
      o[2] = allmax_scalar(v, __dmul_rn(in[(long)p * count + (count > 1 ? 1 : 0)], (double)(1 + (e + p) % P)));
    }
    __syncthreads();
    for (long i = threadIdx.x; i < (long)r * cnt; i += blockDim.x)
      shard[i] = (double)(1000 * e + 10 * p) + 1e-3 * (double)i;
    __syncthreads();
    scatter_body(v, shard, r, cnt, off, full, e & 1, threadIdx.x, blockDim.x);
    __syncthreads();
    barrier_body(v);
    __syncthreads();
  }
}

// gram_with_reinit (engine.hpp:279-296) on a sharded factor.  The factor's
// column c (reference indexing) is row c of the r×full replica; this rank holds
// entries [off, off+cnt) in `local` (r × cnt).  G holds the all-reduced Gram.
// A redraw generates the whole column from mt19937_64(mix_seed(seed, salt,
// attempt)) in the reference order and keeps this rank's slice (stored into
// the local shard and every rank's replica), then the partial Grams are
// recomputed and all-reduced again — all ranks take identical decisions.
__global__ void __launch_bounds__(256) reinit_fixup_dist(const View* vp, double* local, int r, long cnt, long off,
                                                        long full, int which, double* G, uint64_t reinit_seed, int side,
                                                        DevState* st) {
  if (!dev_active(st)) return;
  const View& v = *vp;
  __shared__ int bad[1024];
  __shared__ int nbad;
  const uint64_t salt = 2ULL * st->k + (uint64_t)side;
  for (uint64_t attempt = 0;; ++attempt) {
    if (threadIdx.x == 0) {
      double maxd = 0.0;
      for (int i = 0; i < r; ++i) maxd = (maxd < G[i * r + i]) ? G[i * r + i] : maxd;
      const double fl = __dmul_rn(1e-16, maxd);
      int nb = 0;
      for (int kk = 0; kk < r; ++kk)
        if (!(G[kk * r + kk] > fl) && nb < 1024) bad[nb++] = kk;
      nbad = nb;
    }
    __syncthreads();
    if (nbad == 0) return;
    if (attempt > (uint64_t)r + 2) {
      if (threadIdx.x == 0) {
        st->error_code = ENMF_NO_CONVERGENCE;
        st->active = 0;
      }
      return;
    }
    if (threadIdx.x == 0) {
      DevMt64 gen;
      mt64_seed(gen, mix_seed(reinit_seed, salt, attempt));
      for (int q = 0; q < nbad; ++q) {
        const int c = bad[q];
        for (long i = 0; i < full; ++i) {
          const double u = uniform_unit(gen);
          if (i >= off && i < off + cnt) {
            local[(long)c * cnt + (i - off)] = u;
            for (int p = 0; p < v.world; ++p) {
              double* rep = which == 0 ? v.full_peer_w[p] : v.full_peer_t[p];
              rep[(long)c * full + i] = u;
            }
          }
        }
      }
      st->reinit_events |= 1 << side;
    }
    __syncthreads();
    __shared__ double part[1];
    (void)part;
    // recompute this rank's partial Gram (reference order over the local range)
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
      const int kk = e / r, j = e % r;
      if (kk > j) continue;
      const double* ak = local + (long)kk * cnt;
      const double* aj = local + (long)j * cnt;
      double s = 0.0;
      for (long i = 0; i < cnt; ++i) s = __dadd_rn(s, __dmul_rn(ak[i], aj[i]));
      G[kk * r + j] = s;
      G[j * r + kk] = s;
    }
    __syncthreads();
    allreduce_block(v, G, r * r, G);
  }
}

// Post-BPP checks across ranks: total exchanges (NoConvergence) and NaN flag.
__global__ void bpp_check_dist(const View* v, DevState* st, int side, int r, long Ntotal, unsigned long long* exchanges,
                               int* rounds, int* nonfinite, double* scratch) {
  if (!st || !dev_active(st)) return;
  if (threadIdx.x == 0) {
    scratch[0] = (double)*exchanges;
    scratch[1] = (double)*nonfinite;
  }
  __syncthreads();
  allreduce_block(*v, scratch, 2, scratch);
  if (threadIdx.x == 0) {
    st->bpp_rounds[side] = *rounds;
    st->bpp_exchanges[side] = (unsigned long long)scratch[0];
    if (scratch[0] > 3.0 * (double)r * (double)Ntotal) {
      st->error_code = ENMF_NO_CONVERGENCE;
      st->active = 0;
    } else if (scratch[1] != 0.0) {
      st->error_code = ENMF_NON_FINITE;
      st->active = 0;
    }
    *exchanges = 0;
    *rounds = 0;
    *nonfinite = 0;
  }
}

}  // namespace dist

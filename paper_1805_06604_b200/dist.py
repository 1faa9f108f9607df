"""Multi-GPU (sharded) runs of the hot path — SURVEY §8(e).

One process per GPU.  Rank p of P owns X[:, J_p] (columns, for W_yᵀX) and
X[I_p, :] (rows, for X·Tᵀ), and the shards W[I_p, :], H[:, J_p].  The device
engine exchanges only the factor shards (all-gather into full replicas), the
r×r Gram / error partials (sum all-reduce) and one scalar per HALS sweep, all
through CUDA-IPC peer memory over NVLink (csrc/dist.cuh).  This module does
the one-time host setup: every rank exports the IPC handle of its shared
buffer and the caller's channel (torch.distributed, or any all-gather of
bytes) distributes them.

    ctx = ShardedContext(local_rank, rank, world, m, n, r, torch_exchange())
    ctx.load_sharded_device(x_cols.data_ptr(), x_rows.data_ptr())
    ctx.begin_device(w_shard.data_ptr(), h_shard.data_ptr(), r, cfg)
    ctx.step(K); recs = ctx.sync(); ctx.end(w_out_ptr, h_out_ptr)
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List

import numpy as np

from . import _lib as L
from .enmf import Context, _check, _f64, _p

IPC_HANDLE_BYTES = 64  # sizeof(cudaIpcMemHandle_t)


def shard_bounds(m: int, n: int, rank: int, world: int):
    """(row0, mp, col0, np) of `rank` — balanced contiguous blocks (engine.cu shard_bounds)."""
    vals = [C.c_size_t() for _ in range(4)]
    L.load().enmf_gpu_dist_shard(m, n, rank, world, *[C.byref(v) for v in vals])
    return tuple(int(v.value) for v in vals)


def shard_bounds_py(m: int, n: int, rank: int, world: int):
    """Pure-Python twin of shard_bounds (host logic tests without the library)."""
    def one(length):
        base, extra = divmod(length, world)
        cnt = base + (1 if rank < extra else 0)
        off = rank * base + min(rank, extra)
        return off, cnt
    r0, mp = one(m)
    c0, np_ = one(n)
    return r0, mp, c0, np_


def torch_exchange(group=None) -> Callable[[bytes], List[bytes]]:
    """All-gather of per-rank byte strings over torch.distributed (any backend)."""
    import torch.distributed as dist

    def ex(b: bytes) -> List[bytes]:
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, b, group=group)
        dist.barrier(group)
        return out
    return ex


def exchange_selftest(ctx: Context, world: int, contributions: np.ndarray, epochs: int, r: int, full: int):
    """The exchange primitives of csrc/dist.cuh with `world` ranks on ONE GPU (one cooperative launch,
    block p = rank p; enmf_gpu_dist_selftest).  contributions: (world, count).  Returns (red, sc,
    rep_w, rep_t): red[p, e] = rank p's all-reduced vector of round e (contributions·(e+1) summed in
    rank order), sc[p, e] = (gain sum, flag OR, max), rep_*[p] = rank p's r×full replicas."""
    a = _f64(contributions, "contributions")
    if a.ndim != 2 or a.shape[0] != world:
        raise ValueError("exchange_selftest: contributions must be (world, count)")
    count = a.shape[1]
    red = np.empty((world, epochs, count))
    sc = np.empty((world, epochs, 3))
    rep_w = np.empty((world, r, full))
    rep_t = np.empty((world, r, full))
    _check(ctx._lib.enmf_gpu_dist_selftest(ctx._h, world, count, epochs, r, full, _p(a), _p(red), _p(sc),
                                           _p(rep_w), _p(rep_t)))
    return red, sc, rep_w, rep_t


def hals_solve_vranks(ctx: Context, gram, cross, h0, world: int, max_sweeps: int, stall_fraction: float = 0.01):
    """hals_solve sharded by columns over `world` ranks that all run on ONE GPU in one cooperative
    launch (enmf_gpu_hals_solve_vranks, 64 < r <= 128): the sharded engine's sweep path with its
    per-sweep cross-rank gain exchange.  Returns (H, [sweeps of every rank])."""
    gram, cross, h0 = _f64(gram, "gram"), _f64(cross, "cross"), _f64(h0, "h0")
    r, n = h0.shape
    if cross.shape != (r, n) or gram.shape != (r, r):
        raise ValueError("hals_solve_vranks: shape mismatch")
    h = np.empty_like(h0)
    sw = (C.c_int32 * world)()
    _check(ctx._lib.enmf_gpu_hals_solve_vranks(ctx._h, _p(gram), _p(cross), _p(h0), r, n, world, int(max_sweeps),
                                               float(stall_fraction), _p(h), sw))
    return h, [int(v) for v in sw]


class ShardedContext(Context):
    """An enmf_gpu_ctx in sharded mode (rank `rank` of `world`)."""

    def __init__(self, device: int, rank: int, world: int, m: int, n: int, r: int,
                 exchange: Callable[[bytes], List[bytes]]):
        super().__init__(device)
        self.rank, self.world, self.m, self.n, self.r = rank, world, m, n, r
        self.row0, self.mp, self.col0, self.np = shard_bounds(m, n, rank, world)
        h = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(self._lib.enmf_gpu_dist_alloc(self._h, rank, world, m, n, r, h))
        handles = exchange(bytes(h.raw))
        if len(handles) != world or any(len(x) != IPC_HANDLE_BYTES for x in handles):
            raise RuntimeError("dist: bad handle exchange")
        allh = C.create_string_buffer(b"".join(handles), IPC_HANDLE_BYTES * world)
        _check(self._lib.enmf_gpu_dist_init(self._h, allh))
        exchange(b"\0" * IPC_HANDLE_BYTES)   # barrier: every rank mapped its peers

    def load_sharded_device(self, x_cols_ptr: int, x_rows_ptr: int) -> None:
        _check(self._lib.enmf_gpu_load_dense_sharded(self._h, C.c_void_p(x_cols_ptr), C.c_void_p(x_rows_ptr), 1))

    def load_sharded(self, x_cols, x_rows) -> None:
        xc, xr = _f64(x_cols, "x_cols"), _f64(x_rows, "x_rows")
        if xc.shape != (self.m, self.np) or xr.shape != (self.mp, self.n):
            raise ValueError("load_sharded: block shapes do not match this rank's shard")
        self._keep = (xc, xr)
        _check(self._lib.enmf_gpu_load_dense_sharded(self._h, _p(xc), _p(xr), 0))

    def shard_x(self, x: np.ndarray):
        """This rank's (column block, row block) of a full X."""
        return (np.ascontiguousarray(x[:, self.col0:self.col0 + self.np]),
                np.ascontiguousarray(x[self.row0:self.row0 + self.mp, :]))

    def finalize(self) -> None:
        _check(self._lib.enmf_gpu_dist_finalize(self._h))

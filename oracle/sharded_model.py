"""Sharded restatement of step()/run() for world_size > 1 host-logic tests.

TEST INFRASTRUCTURE ONLY.  A numpy model of exactly the data partition and
exchanges the multi-GPU engine performs (csrc/dist.cuh, engine.cu Layout):
rank p owns X[:, J_p] and X[I_p, :], the shards W[I_p, :] and H[:, J_p], and
only exchanges (a) all-gathers of the W_y / T shards, (b) sums of the r×r
Gram partials and of the fast_error partials, (c) one (gain, nan) pair per
HALS sweep.  Sums are formed by all-gathering the partials and adding them in
rank order, as the device mailbox does, so every rank takes the same
decisions.  tests/test_dist_gloo.py runs it on 2 gloo ranks and checks it
against the C oracle (engine.hpp:309-521 restated in oracle/enmf_oracle.c).

Both inner solvers: HALS (stall rule on the all-reduced gain) and the exact
BPP (per column on the rank's columns, with the WHOLE problem's max|cross| for
the feasibility tolerance and its column count for the exchange limit —
nnls.hpp:271-283 — the quantities the device exchanges in bpp_check_dist), and
the dead-column reinit (engine.hpp:268-296): the Gram diagonal check on the
all-reduced Gram, every rank drawing the full redraw stream of
mt19937_64(mix_seed(seed, salt, attempt)) and keeping its own slice.
"""
from __future__ import annotations

import math

import numpy as np


def shard(length, rank, world):
    base, extra = divmod(length, world)
    cnt = base + (1 if rank < extra else 0)
    off = rank * base + min(rank, extra)
    return off, cnt


class Comm:
    """All-gather / ordered-sum over torch.distributed (gloo)."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def gather(self, a: np.ndarray):
        out = [None] * self.world
        self.dist.all_gather_object(out, np.ascontiguousarray(a))
        return out

    def sum(self, a):
        parts = self.gather(np.asarray(a, dtype=np.float64))
        s = parts[0].copy()
        for q in range(1, self.world):
            s = s + parts[q]
        return s


def hals(comm, G, Cm, H0, max_sweeps, stall):
    """hals_solve (nnls.hpp:154-176) on this rank's columns; the stall test
    uses the gain summed over all ranks."""
    r = G.shape[0]
    H = H0.copy()
    first = 0.0
    sweeps = 0
    while True:
        gain = 0.0
        for k in range(r):
            gkk = G[k, k]
            b = Cm[k] - G[k] @ H + gkk * H[k]
            t = b / gkk
            nxt = np.where(t > 0.0, t, 0.0)
            gain += gkk * float(np.sum((H[k] - t) ** 2 - (nxt - t) ** 2))
            H[k] = nxt
        sweeps += 1
        gain = float(comm.sum(np.array([gain]))[0])
        if sweeps == 1:
            first = gain
        if sweeps >= max_sweeps or gain <= stall * max(first, 0.0):
            return H, sweeps


def _orc():
    from oracle.oracle import Oracle
    return Oracle("port")


def bpp(comm, G, Cm, H0, n_all):
    """active_set_solve on this rank's columns with the global max|C| and column count."""
    import ctypes as C
    orc = _orc()
    fn = orc.lib.orc_active_set_solve_shard
    dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
    fn.argtypes = [dp, dp, dp, C.c_size_t, C.c_size_t, C.c_double, C.c_size_t, dp, C.POINTER(C.c_int32),
                   C.POINTER(C.c_uint64)]
    fn.restype = C.c_int
    cmax = float(np.max(np.abs(Cm))) if Cm.size else 0.0
    cmax = max(float(v[0]) for v in comm.gather(np.array([cmax])))
    r, n = H0.shape
    H = np.zeros((r, n))
    rounds, exch = C.c_int32(), C.c_uint64()
    rc = fn(np.ascontiguousarray(G), np.ascontiguousarray(Cm), np.ascontiguousarray(H0), r, n, cmax, n_all, H,
            C.byref(rounds), C.byref(exch))
    assert rc == 0, rc
    total = int(comm.sum(np.array([float(exch.value)]))[0])
    assert total <= 3 * r * n_all, "NoConvergence (exchange limit)"
    return H


def gram_with_reinit(comm, A, off, total, seed, salt, by_rows):
    """engine.hpp:279-296 on a shard.  A: this rank's slice of the factor whose Gram is formed —
    by_rows: W_y rows (A is mp × r, the columns of W_y have `total` = m entries); otherwise
    T's columns (A is r × np, the rows of T have total = n entries).  Returns (G, A, redrawn)."""
    orc = _orc()
    import ctypes as C
    orc.lib.orc_uniform_stream.argtypes = [C.c_uint64, C.c_size_t,
                                           np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")]
    r = A.shape[1] if by_rows else A.shape[0]
    A = A.copy()
    redrawn = False
    for attempt in range(r + 4):
        G = comm.sum(A.T @ A if by_rows else A @ A.T)
        floor = 1e-16 * max(0.0, float(np.max(np.diag(G))))
        bad = [k for k in range(r) if not (G[k, k] > floor)]
        if not bad:
            return G, A, redrawn
        assert attempt <= r + 2, "NoConvergence (degenerate column persists)"
        stream = np.empty(len(bad) * total)
        orc.lib.orc_uniform_stream(orc.mix_seed(seed, salt, attempt), stream.size, stream)
        cnt = A.shape[0] if by_rows else A.shape[1]
        for q, k in enumerate(bad):
            vals = stream[q * total + off: q * total + off + cnt]
            if by_rows:
                A[:, k] = vals
            else:
                A[k, :] = vals
        redrawn = True
    raise AssertionError("unreachable")


def update_beta(s, dec):
    used = s["beta"]
    if dec:
        s["beta"] = min(s["beta_bar"], s["gamma"] * s["beta"])
        s["beta_bar"] = min(1.0, s["gamma_bar"] * s["beta_bar"])
    else:
        s["beta"] = s["beta"] / s["eta"]
        s["beta_bar"] = s["beta_prev"]
    s["beta_prev"] = used


def run_sharded(comm, X, W0, H0, iters, hp=3, beta0=0.5, gamma=1.01, gamma_bar=1.005, eta=1.5, ratio=0.5,
                stall=0.01, extrapolation=True, inner_h="hals", inner_w="hals", reinit_seed=0, max_sweeps=0):
    """run() (engine.hpp:447-521) on this rank's shards of the full X / W0 / H0 (only the shards
    are read).  Returns (errors, restarted, W shard, H shard, ||X||, reinit events)."""
    m, n = X.shape
    r = W0.shape[1]
    p, P = comm.rank, comm.world
    r0, mp = shard(m, p, P)
    c0, np_ = shard(n, p, P)
    Xc = X[:, c0:c0 + np_]
    Xr = X[r0:r0 + mp, :]
    W = W0[r0:r0 + mp].copy()
    H = H0[:, c0:c0 + np_].copy()
    Wy, Hy = W.copy(), H.copy()
    setup = float(m) * float(n) * float(r)
    ms_h = max_sweeps or 1 + int(math.floor(ratio * setup / (float(n) * r * r)))
    ms_w = max_sweeps or 1 + int(math.floor(ratio * setup / (float(m) * r * r)))
    nx2 = float(comm.sum(np.array([np.sum(Xr * Xr)]))[0])
    nx = math.sqrt(nx2)

    def err(Wn, Pm, GW):
        dot = float(comm.sum(np.array([np.sum(Wn * Pm)]))[0])
        gwn = comm.sum(Wn.T @ Wn)
        v = nx2 - 2.0 * dot + float(np.sum(gwn * GW))
        return math.sqrt(max(0.0, v))

    def solve(kind, G, Cm, H0_, n_all, ms):
        return bpp(comm, G, Cm, H0_, n_all) if kind == "exact" else hals(comm, G, Cm, H0_, ms, stall)[0]

    GW = comm.sum(H @ H.T)
    Hfull = np.concatenate(comm.gather(H), axis=1)
    e_prev = err(W, Xr @ Hfull.T, GW)
    errors, restarted, reinit = [e_prev], [0], [0]
    sch = dict(beta=beta0, beta_bar=1.0, beta_prev=beta0, gamma=gamma, gamma_bar=gamma_bar, eta=eta)
    for k in range(1, iters + 1):
        beta = sch["beta"] if extrapolation else 0.0
        ev = 0
        GH, Wy, red = gram_with_reinit(comm, Wy, r0, m, reinit_seed, 2 * k, True)
        ev |= 1 if red else 0
        Wyfull = np.concatenate(comm.gather(Wy), axis=0)
        CH = Wyfull.T @ Xc
        Hn = solve(inner_h, GH, CH, Hy, n, ms_h)
        if hp >= 2:
            Hy = Hn + beta * (Hn - H) if extrapolation else Hn.copy()
            if hp == 3:
                Hy = np.where(Hy > 0.0, Hy, 0.0)
        T = Hy if hp >= 2 else Hn
        GW, T, red = gram_with_reinit(comm, T, c0, n, reinit_seed, 2 * k + 1, False)
        if red:
            ev |= 2
            if hp >= 2:
                Hy = T
            else:
                Hn = T
        Tfull = np.concatenate(comm.gather(T), axis=1)
        Pm = Xr @ Tfull.T
        WnT = solve(inner_w, GW, Pm.T.copy(), Wy.T.copy(), m, ms_w)
        Wn = WnT.T.copy()
        Wy = Wn + beta * (Wn - W) if extrapolation else Wn.copy()
        if hp == 1:
            Hy = Hn + beta * (Hn - H) if extrapolation else Hn.copy()
        e = err(Wn, Pm, GW)
        if e > e_prev:
            Wy, Hy = W.copy(), H.copy()
            restarted.append(1)
        else:
            W, H = Wn, Hn
            restarted.append(0)
        if extrapolation:
            update_beta(sch, e <= e_prev)
        e_prev = e
        errors.append(e)
        reinit.append(ev)
    return np.array(errors), np.array(restarted), W, H, nx, np.array(reinit)

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
HALS only (the inner solver of the headline config); no column reinit.
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
                stall=0.01, extrapolation=True):
    """E-A-HALS run() on this rank's shards of the full X / W0 / H0 (only the
    shards are read).  Returns (errors, restarted, W shard, H shard)."""
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
    ms_h = 1 + int(math.floor(ratio * setup / (float(n) * r * r)))
    ms_w = 1 + int(math.floor(ratio * setup / (float(m) * r * r)))
    nx2 = float(comm.sum(np.array([np.sum(Xr * Xr)]))[0])
    nx = math.sqrt(nx2)

    def err(Wn, Pm, GW):
        dot = float(comm.sum(np.array([np.sum(Wn * Pm)]))[0])
        gwn = comm.sum(Wn.T @ Wn)
        v = nx2 - 2.0 * dot + float(np.sum(gwn * GW))
        return math.sqrt(max(0.0, v))

    GW = comm.sum(H @ H.T)
    Hfull = np.concatenate(comm.gather(H), axis=1)
    e_prev = err(W, Xr @ Hfull.T, GW)
    errors, restarted = [e_prev], [0]
    sch = dict(beta=beta0, beta_bar=1.0, beta_prev=beta0, gamma=gamma, gamma_bar=gamma_bar, eta=eta)
    for _ in range(iters):
        beta = sch["beta"] if extrapolation else 0.0
        Wyfull = np.concatenate(comm.gather(Wy), axis=0)
        GH = comm.sum(Wy.T @ Wy)
        CH = Wyfull.T @ Xc
        Hn, _ = hals(comm, GH, CH, Hy, ms_h, stall)
        if hp >= 2:
            Hy = Hn + beta * (Hn - H) if extrapolation else Hn.copy()
            if hp == 3:
                Hy = np.where(Hy > 0.0, Hy, 0.0)
        T = Hy if hp >= 2 else Hn
        Tfull = np.concatenate(comm.gather(T), axis=1)
        GW = comm.sum(T @ T.T)
        Pm = Xr @ Tfull.T
        WnT, _ = hals(comm, GW, Pm.T.copy(), Wy.T.copy(), ms_w, stall)
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
    return np.array(errors), np.array(restarted), W, H, nx

"""CPU tier, world_size 2 and 3 (gloo): the multi-GPU partition and exchanges.

The device engine's sharding (csrc/dist.cuh, engine.cu Layout) is modelled in
oracle/sharded_model.py with the same data partition and the same exchanged
quantities; gloo ranks run it and the result must match the single-process
oracle / the reference's fixtures: identical restart sequence, errors within
1e-9 relative, and the gathered factors within 1e-6 — i.e. the sharded algorithm
is the reference's — for E-A-HALS, E-ANLS (sharded BPP with the global max|C|
and exchange limit) and the dead-column reinit (every rank drawing the full
redraw stream, keeping its slice); every rank's decision words (errors, restart
flags, reinit events) are compared across ranks.  Also checks the shard bounds
the library uses.

Why not the device engine at world 2 here: the pool gives one GPU per call, and
ranks whose kernels wait on one another (the per-sweep gain exchange inside the
persistent sweep kernel, the peer-memory mailboxes) must not run as separate
launches on one GPU (B200_PROFILING.md: Xid 109 context-switch timeouts).  The
device exchange kernels run at world 1 on the B200
(tests/test_gpu_parity.py::test_sharded_engine_world1_matches_single).
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, x, w0, h0, iters, kw):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.sharded_model import Comm, run_sharded
        comm = Comm()
        errors, restarted, W, H, nx, reinit = run_sharded(comm, x, w0, h0, iters, **kw)
        Ws = comm.gather(W)
        Hs = comm.gather(H)
        words = comm.gather(np.concatenate([errors, restarted, reinit]))   # every rank's decisions
        if rank == 0:
            q.put((errors, restarted, np.concatenate(Ws, axis=0), np.concatenate(Hs, axis=1), nx, reinit, words))
    finally:
        dist.destroy_process_group()


def _run_world(world, x, w0, h0, iters, **kw):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pt = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, pt, q, x, w0, h0, iters, kw)) for k in range(world)]
    for p_ in procs:
        p_.start()
    out = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    words = out[-1]
    for w_ in words[1:]:
        assert np.array_equal(w_, words[0]), "ranks took different decisions"
    return out[:-1]


def _check(out, err_ref, restarted_ref, wr, hr, nxr):
    errors, restarted, W, H, nx, _ = out
    assert abs(nx - nxr) <= 1e-12 * nxr
    assert np.array_equal(restarted, np.asarray(restarted_ref))
    assert np.max(np.abs(errors - err_ref) / err_ref) <= 1e-9
    assert np.max(np.abs(W - wr)) <= 1e-6 * np.max(np.abs(wr))
    assert np.max(np.abs(H - hr)) <= 1e-6 * np.max(np.abs(hr))


@pytest.mark.parametrize("hp", [3, 1])
def test_sharded_model_matches_oracle_world2(port, hp):
    from oracle.oracle import preset
    rng = np.random.default_rng(7)
    m, n, r = 61, 47, 5
    x = rng.random((m, r)) @ rng.random((r, n)) + 0.01 * np.abs(rng.standard_normal((m, n)))
    w0, h0 = port.random_init(m, n, r, 3)
    iters = 25
    ref, wr, hr, nxr = port.run_dense(x, w0, h0, preset(f"e-ahals-hp{hp}", max_outer_iterations=iters))
    _check(_run_world(2, x, w0, h0, iters, hp=hp), ref["error"], ref["restarted"], wr, hr, nxr)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_eanls_matches_oracle(port, world):
    """E-ANLS hp1 (BPP both sides, nnls.hpp:259-406) on a noisy C3-like problem."""
    from oracle.oracle import preset
    rng = np.random.default_rng(17)
    m, n, r = 70, 53, 6
    x = rng.random((m, r)) @ rng.random((r, n))
    x = np.maximum(x + 0.05 * x.mean() * rng.standard_normal((m, n)), 0.0)
    w0, h0 = port.random_init(m, n, r, 4)
    iters = 15
    ref, wr, hr, nxr = port.run_dense(x, w0, h0, preset("e-anls-hp1", max_outer_iterations=iters))
    out = _run_world(world, x, w0, h0, iters, hp=1, beta0=0.5, gamma=1.1, gamma_bar=1.05, eta=1.5,
                     inner_h="exact", inner_w="exact")
    _check(out, ref["error"], ref["restarted"], wr, hr, nxr)


@pytest.mark.parametrize("tag", ["reinit_hals", "reinit_exact"])
def test_sharded_reinit_matches_reference_fixture(golden, tag):
    """The dead-column reinit cases of the reference's own fixtures (engine.hpp:268-296) at world 2:
    the redraw happens on both ranks in the same iteration and the trajectory is the reference's."""
    inp = golden.load("reinit_inputs")
    g = golden.load(tag)
    meta = golden.meta[tag]
    kind = "exact" if meta["inner_h"] == 0 else "hals"
    out = _run_world(2, inp["x"], inp["w0"], inp["h0"], meta["max_outer_iterations"], hp=meta["hp"],
                     beta0=meta["beta0"], gamma=meta["gamma"], gamma_bar=meta["gamma_bar"], eta=meta["eta"],
                     inner_h=kind, inner_w=kind, reinit_seed=meta["reinit_seed"])
    assert out[5][1] & 1, "the W_y column reinit of iteration 1"
    _check(out, g["error"], g["restarted"], g["w"], g["h"], float(g["norm_x"]))


def test_shard_bounds_cover_and_balance():
    from paper_1805_06604_b200.dist import shard_bounds_py
    for m, n, world in [(10, 7, 3), (32768, 32768, 8), (5, 9, 4), (100, 3, 3)]:
        rows, cols = [], []
        for p in range(world):
            r0, mp_, c0, np_ = shard_bounds_py(m, n, p, world)
            rows.append((r0, mp_))
            cols.append((c0, np_))
        assert rows[0][0] == 0 and sum(c for _, c in rows) == m
        assert cols[0][0] == 0 and sum(c for _, c in cols) == n
        for (a, b), (c, _) in zip(rows, rows[1:]):
            assert a + b == c
        assert max(c for _, c in rows) - min(c for _, c in rows) <= 1


def test_shard_bounds_match_library():
    from paper_1805_06604_b200.dist import shard_bounds, shard_bounds_py
    for args in [(10, 7, 1, 3), (32768, 32768, 5, 8), (5, 9, 3, 4)]:
        assert shard_bounds(*args) == shard_bounds_py(*args)

"""CPU tier, world_size 2 (gloo): the multi-GPU partition and exchanges.

The device engine's sharding (csrc/dist.cuh, engine.cu Layout) is modelled in
oracle/sharded_model.py with the same data partition and the same exchanged
quantities; two gloo ranks run it and the result must match the single-process
oracle: identical restart sequence, errors within 1e-9 relative, and the
gathered factors within 1e-6 — i.e. the sharded algorithm is the reference's.
Also checks the shard bounds the library uses.
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


def _worker(rank, world, port, q, x, w0, h0, iters, hp):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.sharded_model import Comm, run_sharded
        comm = Comm()
        errors, restarted, W, H, nx = run_sharded(comm, x, w0, h0, iters, hp=hp)
        Ws = comm.gather(W)
        Hs = comm.gather(H)
        if rank == 0:
            q.put((errors, restarted, np.concatenate(Ws, axis=0), np.concatenate(Hs, axis=1), nx))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("hp", [3, 1])
def test_sharded_model_matches_oracle_world2(port, hp):
    import torch.multiprocessing as mp
    from oracle.oracle import preset
    rng = np.random.default_rng(7)
    m, n, r = 61, 47, 5
    x = rng.random((m, r)) @ rng.random((r, n)) + 0.01 * np.abs(rng.standard_normal((m, n)))
    w0, h0 = port.random_init(m, n, r, 3)
    iters = 25
    ref, wr, hr, nxr = port.run_dense(x, w0, h0, preset(f"e-ahals-hp{hp}", max_outer_iterations=iters))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pt = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, pt, q, x, w0, h0, iters, hp)) for k in range(2)]
    for p_ in procs:
        p_.start()
    errors, restarted, W, H, nx = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert abs(nx - nxr) <= 1e-12 * nxr
    assert np.array_equal(restarted, ref["restarted"])
    assert np.max(np.abs(errors - ref["error"]) / ref["error"]) <= 1e-9
    assert np.max(np.abs(W - wr)) <= 1e-6 * np.max(np.abs(wr))
    assert np.max(np.abs(H - hr)) <= 1e-6 * np.max(np.abs(hr))


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

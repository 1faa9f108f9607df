"""GPU tier: the cross-rank exchange primitives of csrc/dist.cuh executed with
2..8 ranks on the one GPU a call gets — as ONE cooperative launch whose block p plays rank p
(all ranks co-resident, so the epoch-flag spin-waits always make progress; separate processes or
launches that wait on one another must not share a GPU, B200_PROFILING.md).  Same device code
as the sharded engine's kernels: signal_and_wait, the double-buffered mailbox slots,
allreduce_block / allreduce_gain / allmax_scalar, the shard all-gather and its barrier.
Checked: every rank ends every round with the rank-ordered sum, bit for bit (what makes all
ranks take identical β / restart / stall decisions), over enough rounds to reuse both slot
parities many times; the replicas hold every rank's last shard."""
import numpy as np
import pytest

import paper_1805_06604_b200 as E
from paper_1805_06604_b200 import dist as D

pytestmark = pytest.mark.gpu


def _ordered_sum(a):
    s = a[0].copy()
    for q in range(1, a.shape[0]):
        s = s + a[q]
    return s


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_exchange_primitives_world_n_on_one_gpu(ctx, world):
    rng = np.random.default_rng(world)
    count, epochs, r, full = 128 * 128 + 16, 9, 5, 53
    a = rng.standard_normal((world, count)) * np.exp(rng.uniform(-20, 20, (world, count)))
    red, sc, rep_w, rep_t = D.exchange_selftest(ctx, world, a, epochs, r, full)
    for e in range(epochs):
        want = _ordered_sum(a * float(e + 1))
        for p in range(world):
            assert np.array_equal(red[p, e], want), (world, e, p)
        g = _ordered_sum(a[:, 0:1] * float(e + 2))[0]
        mx = max(a[p, 1] * float(1 + (e + p) % world) for p in range(world))
        for p in range(world):
            assert sc[p, e, 0] == g and sc[p, e, 1] == 1.0 and sc[p, e, 2] == mx, (world, e, p)
    # replicas: W holds the last even round's shards, T the last odd round's, of every rank
    base, extra = divmod(full, world)
    for which, rep in ((0, rep_w), (1, rep_t)):
        e = max(x for x in range(epochs) if x % 2 == which)
        want = np.empty((r, full))
        for p in range(world):
            cnt = base + (1 if p < extra else 0)
            off = p * base + min(p, extra)
            want[:, off:off + cnt] = (1000.0 * e + 10.0 * p) + 1e-3 * np.arange(r * cnt).reshape(r, cnt)
        for p in range(world):
            assert np.array_equal(rep[p], want), (world, which, p)


@pytest.mark.parametrize("world,r,n", [(2, 128, 3000), (4, 100, 2222), (3, 72, 1000), (8, 128, 4099)])
def test_sharded_hals_sweeps_world_n_on_one_gpu(ctx, world, r, n):
    """The sharded sweep path of the headline kernel (hals::sweep_tm with grid_decision's cross-rank
    gain exchange, dist::allreduce_gain) with 2-8 ranks co-resident in one cooperative launch
    (sweep_tm<128, true>): every rank stops after the same sweep, which is the single-GPU solve's, and the
    column shards put together are the single-GPU H bit for bit (columns are independent within a
    sweep, nnls.hpp:111-136; only the stall rule couples them)."""
    rng = np.random.default_rng(world * 1000 + r)
    w = rng.random((300, r))
    g = w.T @ w
    c = w.T @ rng.random((300, n))
    h0 = rng.random((r, n))
    for max_sweeps, stall in ((200, 0.01), (7, 1e-300)):
        h1, s1 = ctx.hals_solve(g, c, h0, max_sweeps, stall)
        hv, sv = D.hals_solve_vranks(ctx, g, c, h0, world, max_sweeps, stall)
        assert sv == [s1] * world, (sv, s1)
        assert np.array_equal(hv, h1)

"""The INT8-digit cross-product scheme of csrc/ozaki.cuh restated in numpy (CPU, no GPU):
full 8-bit digits with offsets, the exact rank-one offset corrections, and the truncation-bias
estimate.  Checks the algebra the CUDA path relies on — the int8 digit products plus the
corrections reproduce the offset-digit products exactly, the cuts are exact — and that 6 levels
with the bias estimate land well inside the FP64 accumulation error of the reference's own
product (linalg.hpp:67-124) on C5-like data."""
import math

import numpy as np

S_MAX = 7


def two_prod(a, b):
    """Dekker's error-free product (numpy, elementwise): a·b = p + e exactly."""
    sp = 134217729.0                           # 2^27 + 1
    p = a * b
    ta, tb = sp * a, sp * b
    ah, bh = ta - (ta - a), tb - (tb - b)
    al, bl = a - ah, b - bh
    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return p, e


def exact_product(a, b):
    """a (R×K) · b (K×N), every entry the correctly rounded exact dot product."""
    out = np.empty((a.shape[0], b.shape[1]))
    for i in range(a.shape[0]):
        p, e = two_prod(a[i][:, None], b)
        for j in range(b.shape[1]):
            out[i, j] = math.fsum(np.concatenate([p[:, j], e[:, j]]))
    return out


def cut8(z):
    """ozaki::cut8: z in (-1/2, 1/2) -> D_0 = floor(256 z) in [-128, 127], D_p = floor(256 r) in
    [0, 255] (p >= 1); returns the stored int8 digits d (d_0 = D_0, d_p = D_p - 128)."""
    t = z * 256.0
    d = np.floor(t)
    digs = [d.astype(np.int64)]
    t = t - d
    for _ in range(1, S_MAX):
        t = t * 256.0
        d = np.floor(t)
        t = t - d
        digs.append(d.astype(np.int64) - 128)
    return np.stack(digs)                     # (S_MAX, ...)


def exp_above(mx):
    return np.where(mx > 0, np.frexp(mx)[1], 0)


def digit_product(a, b, S, bias=True):
    """a (R×K) · b (K×N) the way ozaki_cross computes it: rows of a scaled by 2^-(e_i+1),
    columns of b by 2^-(e_j+1) (b scaled per column, the W_yᵀX case)."""
    ea = exp_above(np.max(np.abs(a), axis=1))
    eb = exp_above(np.max(np.abs(b), axis=0))
    da = cut8(a * np.ldexp(1.0, -(ea + 1))[:, None])          # (S_MAX, R, K)
    db = cut8(b * np.ldexp(1.0, -(eb + 1))[None, :])          # (S_MAX, K, N)
    K = a.shape[1]
    asum = da.sum(axis=2)                                     # (S_MAX, R): row sums of d^A_p
    bsum = db.sum(axis=1)                                     # (S_MAX, N): column sums of d^B_q
    c = np.array([0] + [128] * (S_MAX - 1), dtype=np.int64)
    out = np.zeros((a.shape[0], b.shape[1]))
    base = (ea[:, None] + 1) + (eb[None, :] + 1)
    if bias:
        ra = asum + c[:, None] * K
        cb = bsum + c[:, None] * K
        corr = np.zeros_like(out)
        for p in range(1, S):
            for q in range(S - p, S):
                corr += np.ldexp(np.outer(ra[p], cb[q]).astype(np.float64), -8 * (p + q + 2))
        corr /= K
        sa = sum(np.ldexp(ra[p].astype(np.float64), -8 * (p + 1)) for p in range(S))
        sb = sum(np.ldexp(cb[p].astype(np.float64), -8 * (p + 1)) for p in range(S))
        corr += np.ldexp(sa[:, None] + sb[None, :], -8 * S - 1)
        out = np.ldexp(corr, base)
    for w in range(S - 1, -1, -1):
        part = np.zeros(out.shape, dtype=np.int64)
        for q in range(w + 1):
            p = w - q
            g = da[p] @ db[q]                                  # the int8 digit GEMM (exact int32)
            part += g + c[q] * asum[p][:, None] + c[p] * bsum[q][None, :] + c[p] * c[q] * K
        out += np.ldexp(part.astype(np.float64), base - 8 * (w + 2))
    return out


def test_cuts_are_exact_and_in_int8_range():
    rng = np.random.default_rng(0)
    z = (rng.random(4096) - 0.5) * (1 - 2 ** -40)
    d = cut8(z)
    assert d.min() >= -128 and d.max() <= 127
    D = d + np.array([0] + [128] * (S_MAX - 1))[:, None]
    # 7 digits of 8 bits carry z to 2^-56: the cut itself is exact to that depth
    back = sum(np.ldexp(D[p].astype(np.float64), -8 * (p + 1)) for p in range(S_MAX))
    assert np.max(np.abs(back - z)) <= 2.0 ** -56


def test_offset_corrections_are_exact():
    """D^A_p·D^B_q = d^A_p·d^B_q + c_q·rowsum(d^A_p) + c_p·colsum(d^B_q) + c_p·c_q·K exactly."""
    rng = np.random.default_rng(1)
    a, b = rng.random((16, 300)) - 0.2, rng.random((300, 24))
    da, db = cut8(a / 2 ** (exp_above(np.max(np.abs(a))) + 1)), cut8(b / 2 ** (exp_above(np.max(b)) + 1))
    c = np.array([0] + [128] * (S_MAX - 1))
    K = a.shape[1]
    for p in range(S_MAX):
        for q in range(S_MAX):
            lhs = (da[p] + c[p]) @ (db[q] + c[q])
            rhs = da[p] @ db[q] + c[q] * da[p].sum(1)[:, None] + c[p] * db[q].sum(0)[None, :] + c[p] * c[q] * K
            assert np.array_equal(lhs, rhs)
            assert np.abs(da[p] @ db[q]).max() < 2 ** 31          # int32 GEMM exact


def test_six_levels_with_bias_estimate_on_c5_like_data():
    """Signed factor (W_y is never clamped, engine.hpp:387) against C5-like X: 6 levels with the
    bias estimate are far inside FP64 product accuracy, and the estimate is what gets them there."""
    rng = np.random.default_rng(2)
    K, R, N = 2048, 16, 64
    x = rng.random((K, 8)) @ rng.random((8, N)) + np.abs(0.01 * rng.standard_normal((K, N)))
    w = rng.random((K, R)) - 0.05                              # a few negative entries
    exact = exact_product(np.ascontiguousarray(w.T), x)
    scale = np.abs(w.T) @ np.abs(x)
    e6 = np.max(np.abs(digit_product(w.T, x, 6) - exact) / scale)
    e6_nobias = np.max(np.abs(digit_product(w.T, x, 6, bias=False) - exact) / scale)
    fp64 = np.max(np.abs(w.T @ x - exact) / scale)
    assert e6 < 1e-14, e6
    assert e6 < e6_nobias / 10, (e6, e6_nobias)
    assert e6 <= 10 * max(fp64, 2 ** -52), (e6, fp64)

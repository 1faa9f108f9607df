"""Data formats and synthetic generators — the reference's enmf/data.hpp and rng.hpp.

Everything here runs in the native library (csrc/io.cpp, exported through
include/enmf_gpu.h): Matrix Market and dense-CSV readers that parse on all host
threads, writers with the shortest round-trip number format, the per-run trace CSV,
and the mt19937_64 generators the suites draw data and initial factors from.

    read_matrix_market / write_matrix_market      data.hpp:159-257
    read_dense_csv / write_dense_csv              data.hpp:262-309
    write_run_csv                                 data.hpp:316-326
    format_double                                 data.hpp:101-105
    lowrank_factors / gen_lowrank / gen_fullrank
    random_init / uniform_matrix / mix_seed       data.hpp:58-97, rng.hpp:30-57

Errors raise the reference's exception types: ParseError (with `.line`),
UnsupportedFormat, IoError; a non-finite dense CSV value raises InvalidArgument as
the reference's DenseMatrix constructor does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Sequence, Tuple

import numpy as np

from . import _lib as L
from .enmf import (InvalidArgument, IoError, ParseError, RunRecord, UnsupportedFormat,  # noqa: F401
                   _check)

__all__ = [
    "SparseMatrix", "ParseError", "UnsupportedFormat", "IoError", "format_double",
    "read_matrix_market", "write_matrix_market", "read_dense_csv", "write_dense_csv",
    "write_run_csv", "mix_seed", "uniform_matrix", "lowrank_factors", "gen_lowrank", "gen_tiled",
    "gen_fullrank", "random_init",
]


@dataclass
class SparseMatrix:
    """enmf::SparseMatrix (matrix.hpp:153-258): CSR with 64-bit offsets and column indices."""
    rows: int
    cols: int
    offsets: np.ndarray       # uint64, rows + 1
    col_indices: np.ndarray   # uint64, nnz
    values: np.ndarray        # float64, nnz

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @property
    def shape(self) -> Tuple[int, int]:
        return self.rows, self.cols

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols))
        rows = np.repeat(np.arange(self.rows), np.diff(self.offsets.astype(np.int64)))
        d[rows, self.col_indices.astype(np.int64)] = self.values
        return d

    @staticmethod
    def from_triplets(rows: int, cols: int, entries: Sequence[Tuple[int, int, float]]) -> "SparseMatrix":
        """SparseMatrix::from_triplets (matrix.hpp:168-195)."""
        e = list(entries)
        r = np.array([t[0] for t in e], dtype=np.uint64)
        c = np.array([t[1] for t in e], dtype=np.uint64)
        v = np.array([t[2] for t in e], dtype=np.float64)
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        dup = np.nonzero((r[1:] == r[:-1]) & (c[1:] == c[:-1]))[0]
        if dup.size:
            k = int(dup[0]) + 1
            raise InvalidArgument(f"SparseMatrix: duplicate entry at ({int(r[k])}, {int(c[k])})")
        if r.size and (int(r.max()) >= rows or int(c.max()) >= cols):
            raise InvalidArgument("SparseMatrix: entry index out of bounds")
        off = np.zeros(rows + 1, dtype=np.uint64)
        np.add.at(off, r.astype(np.int64) + 1, 1)
        return SparseMatrix(rows, cols, np.cumsum(off, dtype=np.uint64), c, v)

    @staticmethod
    def from_dense(d) -> "SparseMatrix":
        """SparseMatrix::from_dense (matrix.hpp:196-205): the nonzeros in row-major order."""
        d = np.asarray(d, dtype=np.float64)
        i, j = np.nonzero(d)
        off = np.zeros(d.shape[0] + 1, dtype=np.uint64)
        np.add.at(off, i + 1, 1)
        return SparseMatrix(d.shape[0], d.shape[1], np.cumsum(off, dtype=np.uint64),
                            j.astype(np.uint64), d[i, j].copy())


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def _take(handle) -> "SparseMatrix | np.ndarray":
    lib = L.load()
    rows, cols, nnz, sp = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_int32()
    try:
        lib.enmf_io_matrix_shape(handle, C.byref(rows), C.byref(cols), C.byref(nnz), C.byref(sp))
        m, n, k = rows.value, cols.value, nnz.value
        vals = np.ctypeslib.as_array(lib.enmf_io_matrix_values(handle), (k,)).copy() if k else np.zeros(0)
        if not sp.value:
            return vals.reshape(m, n)
        off = np.ctypeslib.as_array(lib.enmf_io_matrix_offsets(handle), (m + 1,)).copy()
        idx = (np.ctypeslib.as_array(lib.enmf_io_matrix_col_indices(handle), (k,)).copy() if k
               else np.zeros(0, dtype=np.uint64))
        return SparseMatrix(m, n, off, idx, vals)
    finally:
        lib.enmf_io_matrix_free(handle)


def read_matrix_market(path) -> SparseMatrix:
    """enmf::read_matrix_market (data.hpp:159-240)."""
    h = C.c_void_p()
    _check(L.load().enmf_io_read_matrix_market(_path(path), C.byref(h)))
    return _take(h)


def read_dense_csv(path) -> np.ndarray:
    """enmf::read_dense_csv (data.hpp:262-295): a float64 (rows, cols) array."""
    h = C.c_void_p()
    _check(L.load().enmf_io_read_dense_csv(_path(path), C.byref(h)))
    return _take(h)


def write_matrix_market(path, x: SparseMatrix) -> None:
    """enmf::write_matrix_market (data.hpp:242-257)."""
    off = np.ascontiguousarray(x.offsets, dtype=np.uint64)
    idx = np.ascontiguousarray(x.col_indices, dtype=np.uint64)
    val = np.ascontiguousarray(x.values, dtype=np.float64)
    if off.size != x.rows + 1 or (x.rows and int(off[-1]) != val.size) or idx.size != val.size:
        raise InvalidArgument("SparseMatrix: inconsistent compressed storage")
    _check(L.load().enmf_io_write_matrix_market(_path(path), off.ctypes.data, idx.ctypes.data, val.ctypes.data,
                                                x.rows, x.cols))


def write_dense_csv(path, x) -> None:
    """enmf::write_dense_csv (data.hpp:297-309)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise InvalidArgument("write_dense_csv: expected a 2-D matrix")
    _check(L.load().enmf_io_write_dense_csv(_path(path), x.ctypes.data, x.shape[0], x.shape[1]))


def write_run_csv(path, record: RunRecord, e_min: float = 0.0) -> None:
    """enmf::write_run_csv (data.hpp:316-326): iter,elapsed_s,rel_err,E,beta,restarted."""
    its = record.iterations
    arr = (L.CIter * max(1, len(its)))()
    for k, it in enumerate(its):
        arr[k].iteration = it.iteration
        arr[k].elapsed_seconds = it.elapsed_seconds
        arr[k].error = it.error
        arr[k].relative_error = it.relative_error
        arr[k].beta = it.beta
        arr[k].restarted = 1 if it.restarted else 0
    _check(L.load().enmf_io_write_run_csv(_path(path), arr, len(its), float(e_min)))


def format_double(v: float) -> str:
    """enmf::format_double (data.hpp:101-105): std::to_chars shortest round trip."""
    buf = C.create_string_buffer(40)
    n = L.load().enmf_io_format_double(float(v), buf, 40)
    return buf.value[:n].decode()


def mix_seed(base: int, a: int = 0, b: int = 0) -> int:
    """enmf::mix_seed (rng.hpp:36-42)."""
    return int(L.load().enmf_mix_seed(base, a, b))


def uniform_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """enmf::uniform_matrix (rng.hpp:51-57)."""
    x = np.empty((rows, cols)) if rows and cols else np.empty(0)
    _check(L.load().enmf_uniform_matrix(rows, cols, seed, x.ctypes.data))
    return x


def random_init(m: int, n: int, r: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """enmf::random_init (data.hpp:90-97): W (m×r) then H (r×n) from one stream."""
    w = np.empty((m, r)) if m and r else np.empty(0)
    h = np.empty((r, n)) if n and r else np.empty(0)
    _check(L.load().enmf_random_init(m, n, r, seed, w.ctypes.data, h.ctypes.data))
    return w, h


def lowrank_factors(m: int, n: int, r: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """enmf::lowrank_factors (data.hpp:58-70)."""
    w = np.empty((m, r)) if m and r else np.empty(0)
    h = np.empty((r, n)) if n and r else np.empty(0)
    _check(L.load().enmf_lowrank_factors(m, n, r, seed, w.ctypes.data, h.ctypes.data))
    return w, h


def gen_lowrank(m: int, n: int, r: int, seed: int) -> np.ndarray:
    """enmf::gen_lowrank (data.hpp:74-80): X = W·H, rounded as the reference's multiply."""
    x = np.empty((m, n)) if m and n else np.empty(0)
    _check(L.load().enmf_gen_lowrank(m, n, r, seed, x.ctypes.data))
    return x


def gen_tiled(m: int, n: int, r: int, seed: int, rows=None, cols=None, tile: int = 4096) -> np.ndarray:
    """BASELINE configs[4] (C5) data, X = W0·H0 + 0.01·|N(0,1)| on tiles with per-tile streams
    (csrc/io.cpp enmf_gen_tiled): the block rows × cols (slices; default the whole matrix)."""
    r0, r1 = (0, m) if rows is None else (rows.start or 0, rows.stop if rows.stop is not None else m)
    c0, c1 = (0, n) if cols is None else (cols.start or 0, cols.stop if cols.stop is not None else n)
    x = np.empty((r1 - r0, c1 - c0))
    _check(L.load().enmf_gen_tiled(m, n, r, seed, tile, r0, r1 - r0, c0, c1 - c0, x.ctypes.data))
    return x


def gen_fullrank(m: int, n: int, seed: int) -> np.ndarray:
    """enmf::gen_fullrank (data.hpp:84-86)."""
    x = np.empty((m, n)) if m and n else np.empty(0)
    _check(L.load().enmf_gen_fullrank(m, n, seed, x.ctypes.data))
    return x

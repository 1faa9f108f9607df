"""Python mirror of the reference enmf API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference's C++
interface (/root/reference/proj/include/enmf):

  SolverConfig / InnerSolver / TimingMode   engine.hpp:56-58,149-200
  IterationRecord / RunRecord               engine.hpp:216-238
  run(x, w0, h0, cfg, timing)               engine.hpp:447-521
  algorithm_config(name)                    bench.hpp:108-135
  gram, cross_wx, cross_xht, frob_norm_sq   linalg.hpp:49-171
  fast_error                                engine.hpp:121-136
  hals_solve, active_set_solve              nnls.hpp:154-176, 259-406
  update_beta, BetaSchedule                 engine.hpp:63-99

Every computation runs on the GPU through libenmf_gpu.so; nothing here
computes on the CPU (no fallback).  Matrices are numpy float64 row-major.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L


# ---------------------------------------------------------------- exceptions
class InvalidArgument(ValueError):
    """std::invalid_argument"""


class NonFiniteIterate(RuntimeError):
    """enmf::NonFiniteIterate (engine.hpp:51-54)"""


class NoConvergence(RuntimeError):
    """enmf::NoConvergence (nnls.hpp:65-68)"""


class DegenerateColumn(RuntimeError):
    """enmf::DegenerateColumn (nnls.hpp:54-63)"""


class CacheStale(RuntimeError):
    """enmf::CacheStale (engine.hpp:41-44)"""


class DeviceError(RuntimeError):
    """CUDA failure (no reference analogue)."""


class ZeroDirection(RuntimeError):
    """enmf::ZeroDirection (engine.hpp:46-49)"""


class ParseError(RuntimeError):
    """enmf::ParseError (data.hpp:34-43); `line` is 0 when the error has no line."""

    def __init__(self, what: str, line: int = 0):
        super().__init__(what)
        self.line = line


class UnsupportedFormat(RuntimeError):
    """enmf::UnsupportedFormat (data.hpp:45-48)"""


class IoError(RuntimeError):
    """enmf::IoError (data.hpp:50-53)"""


_ERRORS = {
    L.ENMF_INVALID_ARGUMENT: InvalidArgument,
    L.ENMF_NON_FINITE: NonFiniteIterate,
    L.ENMF_NO_CONVERGENCE: NoConvergence,
    L.ENMF_DEGENERATE_COLUMN: DegenerateColumn,
    L.ENMF_CUDA_ERROR: DeviceError,
    L.ENMF_CACHE_STALE: CacheStale,
    L.ENMF_UNSUPPORTED_FORMAT: UnsupportedFormat,
    L.ENMF_IO_ERROR: IoError,
    L.ENMF_ZERO_DIRECTION: ZeroDirection,
}


def _check(rc: int) -> None:
    if rc != L.ENMF_OK:
        lib = L.load()
        msg = lib.enmf_gpu_last_error().decode()
        if rc == L.ENMF_PARSE_ERROR:
            raise ParseError(msg, int(lib.enmf_gpu_last_error_line()))
        raise _ERRORS.get(rc, RuntimeError)(msg)


# ------------------------------------------------------------------ config
class InnerSolver(enum.IntEnum):
    exact = L.ENMF_INNER_EXACT
    hals = L.ENMF_INNER_HALS


class TimingMode(enum.IntEnum):
    wall = L.ENMF_TIMING_WALL
    none = L.ENMF_TIMING_NONE


class Precision(enum.IntEnum):
    fp64 = L.ENMF_PRECISION_FP64              # FP64 product path (DMMA / INT8-digit tensor cores)
    tf32 = L.ENMF_PRECISION_TF32              # variant: cross products on TF32 tensor cores
    fp64_exact = L.ENMF_PRECISION_FP64_EXACT  # bitwise-faithful debug path


@dataclass
class SolverConfig:
    """enmf::SolverConfig (engine.hpp:149-173) plus the device precision."""
    inner_h: InnerSolver = InnerSolver.exact
    inner_w: InnerSolver = InnerSolver.exact
    hp: int = 1
    beta0: float = 0.5
    gamma: float = 1.1
    gamma_bar: float = 1.05
    eta: float = 1.5
    max_outer_iterations: int = 500
    max_seconds: float = math.inf
    extrapolation_enabled: bool = True
    literal_hp1_order: bool = False
    inner_sweep_ratio: float = 0.5
    inner_stall_fraction: float = 0.01
    inner_max_sweeps: Optional[int] = None
    reinit_seed: int = 0
    precision: Precision = Precision.fp64

    def to_c(self, timing: TimingMode = TimingMode.wall) -> L.CConfig:
        if self.inner_max_sweeps is not None and self.inner_max_sweeps < 1:
            raise InvalidArgument("SolverConfig: inner_max_sweeps must be >= 1")
        return L.CConfig(
            inner_h=int(self.inner_h), inner_w=int(self.inner_w), hp=int(self.hp),
            extrapolation_enabled=int(bool(self.extrapolation_enabled)), beta0=self.beta0,
            gamma=self.gamma, gamma_bar=self.gamma_bar, eta=self.eta,
            max_outer_iterations=int(self.max_outer_iterations), max_seconds=float(self.max_seconds),
            literal_hp1_order=int(bool(self.literal_hp1_order)), timing=int(timing),
            inner_sweep_ratio=self.inner_sweep_ratio, inner_stall_fraction=self.inner_stall_fraction,
            inner_max_sweeps=int(self.inner_max_sweeps or 0), reinit_seed=int(self.reinit_seed),
            precision=int(self.precision), reserved=0)

    def validate(self) -> None:
        """SolverConfig::validate (engine.hpp:175-199)."""
        c = self.to_c()
        _check(L.load().enmf_gpu_config_validate(C.byref(c)))


def algorithm_config(name: str) -> SolverConfig:
    """detail::algorithm_config (bench.hpp:108-135)."""
    c = L.CConfig()
    _check(L.load().enmf_gpu_config_preset(C.byref(c), name.encode()))
    return SolverConfig(
        inner_h=InnerSolver(c.inner_h), inner_w=InnerSolver(c.inner_w), hp=c.hp, beta0=c.beta0,
        gamma=c.gamma, gamma_bar=c.gamma_bar, eta=c.eta,
        max_outer_iterations=c.max_outer_iterations, max_seconds=c.max_seconds,
        extrapolation_enabled=bool(c.extrapolation_enabled),
        literal_hp1_order=bool(c.literal_hp1_order), inner_sweep_ratio=c.inner_sweep_ratio,
        inner_stall_fraction=c.inner_stall_fraction, inner_max_sweeps=None,
        reinit_seed=c.reinit_seed)


DEFAULT_ALGORITHMS = ["anls", "e-anls-hp1", "e-anls-hp3", "ahals", "e-ahals-hp1", "e-ahals-hp3"]


@dataclass
class BetaSchedule:
    """enmf::BetaSchedule (engine.hpp:63-82)."""
    beta: float = 0.5
    beta_bar: float = 1.0
    beta_prev: float = 0.5
    gamma: float = 1.1
    gamma_bar: float = 1.05
    eta: float = 1.5


def update_beta(s: BetaSchedule, error_decreased: bool) -> BetaSchedule:
    """update_beta (engine.hpp:88-99) — the same scalar code the device runs."""
    o = L.load().enmf_gpu_update_beta(L.CBeta(**s.__dict__), int(bool(error_decreased)))
    return BetaSchedule(**{k: getattr(o, k) for k, _ in L.CBeta._fields_})


# ----------------------------------------------------------------- records
@dataclass
class IterationRecord:
    iteration: int = 0
    elapsed_seconds: float = 0.0
    error: float = 0.0
    relative_error: float = 0.0
    beta: float = 0.0
    restarted: bool = False
    inner_h_count: int = 0
    inner_w_count: int = 0
    reinit_events: int = 0


@dataclass
class FactorPair:
    w: np.ndarray
    h: np.ndarray


@dataclass
class RunRecord:
    iterations: List[IterationRecord] = field(default_factory=list)
    factors: Optional[FactorPair] = None
    norm_x: float = 0.0

    def final_relative_error(self) -> float:
        return self.iterations[-1].relative_error if self.iterations else 0.0

    # column views used by tests
    def column(self, name: str) -> np.ndarray:
        return np.array([getattr(r, name) for r in self.iterations])


_ITER_DTYPE = np.dtype([("iteration", "<u8"), ("elapsed_seconds", "<f8"), ("error", "<f8"),
                        ("relative_error", "<f8"), ("beta", "<f8"), ("restarted", "<i4"),
                        ("inner_h_count", "<i4"), ("inner_w_count", "<i4"), ("reinit_events", "<i4")])


def _records_np(rows: np.ndarray) -> List[IterationRecord]:
    """IterationRecords from a structured array of enmf_gpu_iter (one tolist() instead of a
    ctypes field access per value)."""
    return [IterationRecord(it, el, e, re, b, rs != 0, ih, iw, ev)
            for it, el, e, re, b, rs, ih, iw, ev in rows.tolist()]


def _records(arr, count) -> List[IterationRecord]:
    """IterationRecords from the first `count` entries of a ctypes array of enmf_gpu_iter."""
    if count == 0:
        return []
    return _records_np(np.frombuffer(arr, dtype=_ITER_DTYPE, count=count))


def _f64(a, name):
    a = np.asarray(a)
    if a.dtype != np.float64:
        a = a.astype(np.float64)
    return np.ascontiguousarray(a)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- context
class Context:
    """One enmf_gpu_ctx (stream + device buffers).  One per thread."""

    def __init__(self, device: int = -1):
        self._lib = L.load()
        h = C.c_void_p()
        _check(self._lib.enmf_gpu_create(C.byref(h), device))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.enmf_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.enmf_gpu_kernel_launches(self._h))

    def set_precision(self, p: Precision) -> None:
        _check(self._lib.enmf_gpu_set_precision(self._h, int(p)))

    # -- run ----------------------------------------------------------------
    def run(self, x, w0, h0, cfg: SolverConfig, timing: TimingMode = TimingMode.wall) -> RunRecord:
        """enmf::run<DenseMatrix> (engine.hpp:447-521)."""
        x, w0, h0 = _f64(x, "x"), _f64(w0, "w0"), _f64(h0, "h0")
        if x.ndim != 2 or w0.ndim != 2 or h0.ndim != 2:
            raise InvalidArgument("run: matrices must be 2-D")
        m, n = x.shape
        r = w0.shape[1]
        if w0.shape[1] != h0.shape[0]:
            raise InvalidArgument("run: factor inner dimensions disagree")
        if w0.shape[0] != m or h0.shape[1] != n:
            raise InvalidArgument("run: factor shapes do not match the data matrix")
        c = cfg.to_c(timing)
        cap = int(cfg.max_outer_iterations) + 1
        iters = (L.CIter * cap)()
        nit = C.c_size_t(0)
        w = np.empty((m, r))
        h = np.empty((r, n))
        nx = C.c_double(0)
        _check(self._lib.enmf_gpu_run_dense(self._h, _p(x), m, n, _p(w0), _p(h0), r, C.byref(c), iters, cap,
                                            C.byref(nit), _p(w), _p(h), C.byref(nx)))
        return RunRecord(_records(iters, min(nit.value, cap)), FactorPair(w, h), nx.value)

    def run_csr(self, offsets, col_idx, vals, m: int, n: int, w0, h0, cfg: SolverConfig,
                timing: TimingMode = TimingMode.wall) -> RunRecord:
        """enmf::run<SparseMatrix> (engine.hpp:447-521 with linalg.hpp:86-104,127-146,167-171).
        offsets (m+1) / col_idx (nnz) as uint64, vals (nnz) float64: the SparseMatrix CSR arrays."""
        self.load_csr(offsets, col_idx, vals, m, n)
        return self._solve_host(w0, h0, m, n, cfg, timing)

    def load_csr(self, offsets, col_idx, vals, m: int, n: int) -> None:
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        ci = np.ascontiguousarray(col_idx, dtype=np.uint64)
        v = _f64(vals, "vals")
        if off.shape != (m + 1,) or ci.shape != v.shape:
            raise InvalidArgument("SparseMatrix: inconsistent compressed storage")
        _check(self._lib.enmf_gpu_load_csr(self._h, off.ctypes.data, ci.ctypes.data, v.ctypes.data, m, n, v.size))

    def _solve_host(self, w0, h0, m, n, cfg: SolverConfig, timing: TimingMode) -> RunRecord:
        w0, h0 = _f64(w0, "w0"), _f64(h0, "h0")
        r = w0.shape[1]
        if w0.shape[1] != h0.shape[0]:
            raise InvalidArgument("run: factor inner dimensions disagree")
        if w0.shape[0] != m or h0.shape[1] != n:
            raise InvalidArgument("run: factor shapes do not match the data matrix")
        c = cfg.to_c(timing)
        cap = int(cfg.max_outer_iterations) + 1
        iters = (L.CIter * cap)()
        nit = C.c_size_t(0)
        w = np.empty((m, r))
        h = np.empty((r, n))
        nx = C.c_double(0)
        _check(self._lib.enmf_gpu_solve(self._h, _p(w0), _p(h0), r, 0, C.byref(c), iters, cap, C.byref(nit),
                                        _p(w), _p(h), C.byref(nx)))
        return RunRecord(_records(iters, min(nit.value, cap)), FactorPair(w, h), nx.value)

    def load_device(self, x_ptr: int, m: int, n: int) -> None:
        """Borrow a device-resident X (e.g. torch.Tensor.data_ptr())."""
        _check(self._lib.enmf_gpu_load_dense(self._h, C.c_void_p(x_ptr), m, n, 1))

    def load(self, x) -> None:
        x = _f64(x, "x")
        _check(self._lib.enmf_gpu_load_dense(self._h, _p(x), x.shape[0], x.shape[1], 0))

    def solve_device(self, w0_ptr: int, h0_ptr: int, r: int, cfg: SolverConfig, w_out_ptr: int = 0,
                     h_out_ptr: int = 0, timing: TimingMode = TimingMode.none) -> RunRecord:
        """Solve on the resident X from device factors (outputs to device pointers)."""
        c = cfg.to_c(timing)
        cap = int(cfg.max_outer_iterations) + 1
        iters = (L.CIter * cap)()
        nit = C.c_size_t(0)
        nx = C.c_double(0)
        _check(self._lib.enmf_gpu_solve(self._h, C.c_void_p(w0_ptr), C.c_void_p(h0_ptr), r, 1, C.byref(c), iters,
                                        cap, C.byref(nit), C.c_void_p(w_out_ptr or None),
                                        C.c_void_p(h_out_ptr or None), C.byref(nx)))
        return RunRecord(_records(iters, min(nit.value, cap)), None, nx.value)

    # -- session: run() split into begin / step / sync / end ------------------
    def begin_device(self, w0_ptr: int, h0_ptr: int, r: int, cfg: SolverConfig,
                     timing: TimingMode = TimingMode.none) -> None:
        c = cfg.to_c(timing)
        self._session_cap = int(cfg.max_outer_iterations) + 1
        _check(self._lib.enmf_gpu_begin(self._h, C.c_void_p(w0_ptr), C.c_void_p(h0_ptr), r, 1, C.byref(c)))

    def begin(self, w0, h0, cfg: SolverConfig, timing: TimingMode = TimingMode.none) -> None:
        w0, h0 = _f64(w0, "w0"), _f64(h0, "h0")
        c = cfg.to_c(timing)
        self._session_cap = int(cfg.max_outer_iterations) + 1
        _check(self._lib.enmf_gpu_begin(self._h, _p(w0), _p(h0), w0.shape[1], 0, C.byref(c)))

    def step(self, count: int = 1) -> None:
        """Enqueue `count` outer iterations (asynchronous)."""
        _check(self._lib.enmf_gpu_step(self._h, int(count)))

    def step_profiled(self) -> dict:
        """One outer iteration with per-phase CUDA-event timings (ms)."""
        out = (C.c_double * 11)()
        _check(self._lib.enmf_gpu_step_profiled(self._h, out, 11))
        keys = ["gram_wy", "cross_wx", "update_h", "extrap_h", "gram_t", "cross_xht", "update_w",
                "error_terms", "decide_finalize", "sweeps_h", "sweeps_w"]
        return dict(zip(keys, list(out)))

    def sync(self) -> List[IterationRecord]:
        cap = getattr(self, "_session_cap", 1)
        iters = (L.CIter * cap)()
        nit = C.c_size_t(0)
        _check(self._lib.enmf_gpu_sync(self._h, iters, cap, C.byref(nit)))
        return _records(iters, min(nit.value, cap))

    def end(self, w_out_ptr: int = 0, h_out_ptr: int = 0) -> float:
        nx = C.c_double(0)
        _check(self._lib.enmf_gpu_end(self._h, C.c_void_p(w_out_ptr or None), C.c_void_p(h_out_ptr or None),
                                      C.byref(nx)))
        return nx.value

    @property
    def stream(self) -> int:
        """cudaStream_t of this context (for torch.cuda.ExternalStream)."""
        return int(self._lib.enmf_gpu_stream(self._h) or 0)

    @property
    def digit_levels(self) -> tuple:
        """(W_yᵀX, X·Tᵀ) digit levels S of the INT8-digit cross products for the loaded X
        (S(S+1)/2 int8 GEMMs per product; 0 = FP64 DMMA GEMM or no X loaded)."""
        lv = (C.c_int32 * 2)()
        _check(self._lib.enmf_gpu_digit_levels(self._h, lv))
        return (lv[0], lv[1])

    # -- kernels --------------------------------------------------------------
    def gram(self, a) -> np.ndarray:
        a = _f64(a, "a")
        g = np.empty((a.shape[1], a.shape[1]))
        _check(self._lib.enmf_gpu_gram(self._h, _p(a), a.shape[0], a.shape[1], _p(g)))
        return g

    def cross_wx(self, w, x) -> np.ndarray:
        w, x = _f64(w, "w"), _f64(x, "x")
        if w.shape[0] != x.shape[0]:
            raise InvalidArgument("cross_wx: row count mismatch")
        out = np.empty((w.shape[1], x.shape[1]))
        _check(self._lib.enmf_gpu_cross_wx(self._h, _p(w), _p(x), x.shape[0], x.shape[1], w.shape[1], _p(out)))
        return out

    def cross_xht(self, x, h) -> np.ndarray:
        x, h = _f64(x, "x"), _f64(h, "h")
        if x.shape[1] != h.shape[1]:
            raise InvalidArgument("cross_xht: column count mismatch")
        out = np.empty((x.shape[0], h.shape[0]))
        _check(self._lib.enmf_gpu_cross_xht(self._h, _p(x), _p(h), x.shape[0], x.shape[1], h.shape[0], _p(out)))
        return out

    def frob_norm_sq(self, x) -> float:
        x = _f64(x, "x")
        v = C.c_double()
        _check(self._lib.enmf_gpu_frob_norm_sq(self._h, _p(x), x.size, C.byref(v)))
        return v.value

    def fast_error(self, norm_x_sq, w, xht, hht) -> float:
        w, xht, hht = _f64(w, "w"), _f64(xht, "xht"), _f64(hht, "hht")
        if w.shape != xht.shape or hht.shape != (w.shape[1], w.shape[1]):
            raise InvalidArgument("fast_error: shape mismatch")
        v = C.c_double()
        _check(self._lib.enmf_gpu_fast_error(self._h, float(norm_x_sq), _p(w), _p(xht), _p(hht), w.shape[0],
                                             w.shape[1], C.byref(v)))
        return v.value

    def hals_solve(self, gram, cross, h0, max_sweeps: int, stall_fraction: float = 0.01):
        gram, cross, h0 = _f64(gram, "gram"), _f64(cross, "cross"), _f64(h0, "h0")
        r, n = h0.shape
        if cross.shape != (r, n) or gram.shape != (r, r):
            raise InvalidArgument("hals_solve: warm start shape mismatch")
        h = np.empty_like(h0)
        sw = C.c_int32()
        _check(self._lib.enmf_gpu_hals_solve(self._h, _p(gram), _p(cross), _p(h0), r, n, int(max_sweeps),
                                             float(stall_fraction), _p(h), C.byref(sw)))
        return h, sw.value

    def optimal_beta_linesearch(self, x, w_n, w, h_y) -> float:
        """enmf::optimal_beta_linesearch (engine.hpp:522-540); x dense or a data.SparseMatrix."""
        w_n, w, h_y = _f64(w_n, "w_n"), _f64(w, "w"), _f64(h_y, "h_y")
        m, r = w_n.shape
        n = h_y.shape[1]
        if w.shape != (m, r) or h_y.shape[0] != r:
            raise InvalidArgument("optimal_beta_linesearch: shape mismatch")
        beta = C.c_double(0)
        if hasattr(x, "offsets"):
            if (x.rows, x.cols) != (m, n):
                raise InvalidArgument("optimal_beta_linesearch: shape mismatch")
            off = np.ascontiguousarray(x.offsets, dtype=np.uint64)
            idx = np.ascontiguousarray(x.col_indices, dtype=np.uint64)
            val = _f64(x.values, "vals")
            _check(self._lib.enmf_gpu_optimal_beta_linesearch_csr(self._h, off.ctypes.data, idx.ctypes.data,
                                                                  val.ctypes.data, m, n, val.size, _p(w_n), _p(w),
                                                                  _p(h_y), r, C.byref(beta)))
        else:
            x = _f64(x, "x")
            if x.shape != (m, n):
                raise InvalidArgument("optimal_beta_linesearch: shape mismatch")
            _check(self._lib.enmf_gpu_optimal_beta_linesearch(self._h, _p(x), m, n, _p(w_n), _p(w), _p(h_y), r,
                                                              C.byref(beta)))
        return beta.value

    def active_set_solve(self, gram, cross, h0):
        gram, cross, h0 = _f64(gram, "gram"), _f64(cross, "cross"), _f64(h0, "h0")
        r, n = h0.shape
        if cross.shape != (r, n) or gram.shape != (r, r):
            raise InvalidArgument("active_set_solve: warm start shape mismatch")
        h = np.empty_like(h0)
        rd = C.c_int32()
        _check(self._lib.enmf_gpu_active_set_solve(self._h, _p(gram), _p(cross), _p(h0), r, n, _p(h),
                                                   C.byref(rd)))
        return h, rd.value


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = _tls.ctx = Context()
    return ctx


def run(x, w0, h0, cfg: SolverConfig, timing: TimingMode = TimingMode.wall) -> RunRecord:
    """enmf::run (engine.hpp:447-521) on the calling thread's GPU context."""
    return default_context().run(x, w0, h0, cfg, timing)


def batch_eligible(m: int, n: int, r: int, cfg: SolverConfig, timing: TimingMode = TimingMode.none) -> bool:
    """Whether runs of this shape and config fit the packed one-CTA-per-run kernel (batch.cuh):
    FP64 (HALS or BPP inner solvers), r <= 32, max(m, n)·(r rounded up to 8) <= 9216, no wall budget, no timing
    records."""
    if timing != TimingMode.none:
        return False
    c = cfg.to_c(timing)
    return L.load().enmf_gpu_batch_eligible(m, n, r, C.byref(c)) == L.ENMF_OK


def run_batch_packed(problems, cfg: SolverConfig, device: int = -1, raise_errors: bool = True) -> List[RunRecord]:
    """Many independent runs of one shape in ONE launch (csrc/batch.cuh): one CTA per run
    executes every step() of enmf::run (engine.hpp:447-521) for its problem.  The FP64 product
    arithmetic of the engine (parity bars, not bit equality).  raise_errors: raise the first
    failing run's error as `run` would; otherwise that run's slot holds the exception."""
    problems = [(_f64(x, "x"), _f64(w0, "w0"), _f64(h0, "h0")) for x, w0, h0 in problems]
    if not problems:
        return []
    m, n = problems[0][0].shape
    r = problems[0][1].shape[1]
    for x, w0, h0 in problems:
        if x.shape != (m, n) or w0.shape != (m, r) or h0.shape != (r, n):
            raise InvalidArgument("run_batch_packed: every problem must have the same shapes")
    B = len(problems)
    xs = np.ascontiguousarray(np.stack([p[0] for p in problems]))
    ws = np.ascontiguousarray(np.stack([p[1] for p in problems]))
    hs = np.ascontiguousarray(np.stack([p[2] for p in problems]))
    c = cfg.to_c(TimingMode.none)
    cap = int(cfg.max_outer_iterations) + 1
    iters = (L.CIter * (cap * B))()
    nit = np.zeros(B, dtype=np.int32)
    st = np.zeros(B, dtype=np.int32)
    wo = np.empty((B, m, r))
    ho = np.empty((B, r, n))
    nx = np.empty(B)
    ctx = default_context() if device < 0 else Context(device)
    ip = C.POINTER(C.c_int32)
    _check(L.load().enmf_gpu_run_batch_dense(ctx._h, B, _p(xs), m, n, _p(ws), _p(hs), r, C.byref(c), iters, cap,
                                             nit.ctypes.data_as(ip), st.ctypes.data_as(ip), _p(wo), _p(ho),
                                             _p(nx)))
    allrec = np.frombuffer(iters, dtype=_ITER_DTYPE, count=cap * B).reshape(B, cap)
    out = []
    for b in range(B):
        if st[b] != L.ENMF_OK:
            err = _ERRORS.get(int(st[b]), RuntimeError)(f"run_batch_packed: run {b} failed (status {int(st[b])})")
            if raise_errors:
                raise err
            out.append(err)
            continue
        recs = _records_np(allrec[b, :min(int(nit[b]), cap)])
        out.append(RunRecord(recs, FactorPair(wo[b], ho[b]), float(nx[b])))
    return out


def run_batch(problems, cfg: SolverConfig, timing: TimingMode = TimingMode.none, streams: int = 8,
              device: int = -1, backend: str = "auto") -> List[RunRecord]:
    """Many independent dense runs in flight together — the paper protocol's dataset × init
    grid that the reference runs on a host thread pool (run_suite, bench.hpp:233-294).

    backend "packed" (the default for eligible batches: same shapes, FP64, r <= 32, small
    problems — batch_eligible): one launch, one CTA per run (run_batch_packed).
    backend "streams": up to `streams` contexts, each with its own CUDA stream and iteration
    graph, take a problem each; all K iterations of every context are enqueued before any
    result is read.  Every run is then computed exactly as `run` computes it on its own (this
    is the path for fp64_exact and large problems)."""
    problems = list(problems)
    if backend not in ("auto", "packed", "streams"):
        raise InvalidArgument("run_batch: backend must be auto, packed or streams")
    if backend != "streams" and problems:
        x0, w00 = problems[0][0], problems[0][1]
        same = all(np.shape(p[0]) == np.shape(x0) and np.shape(p[1]) == np.shape(w00) for p in problems)
        ok = same and np.ndim(x0) == 2 and batch_eligible(np.shape(x0)[0], np.shape(x0)[1], np.shape(w00)[1], cfg,
                                                          timing)
        if ok:
            return run_batch_packed(problems, cfg, device)
        if backend == "packed":
            raise InvalidArgument("run_batch: this batch does not fit the packed kernel (batch_eligible)")
    pool = [Context(device) for _ in range(max(1, min(streams, len(problems))))]
    out: List[RunRecord] = []
    try:
        for start in range(0, len(problems), len(pool)):
            chunk = problems[start:start + len(pool)]
            live = []
            for ctx, (x, w0, h0) in zip(pool, chunk):
                x, w0, h0 = _f64(x, "x"), _f64(w0, "w0"), _f64(h0, "h0")
                if w0.shape[0] != x.shape[0] or h0.shape[1] != x.shape[1] or w0.shape[1] != h0.shape[0]:
                    raise InvalidArgument("run: factor shapes do not match the data matrix")
                ctx.load(x)
                ctx.begin(w0, h0, cfg, timing)
                ctx.step(int(cfg.max_outer_iterations))
                live.append((ctx, x.shape, w0.shape[1]))
            for ctx, (m, n), r in live:
                recs = ctx.sync()
                w = np.empty((m, r))
                h = np.empty((r, n))
                nx = ctx.end(w.ctypes.data, h.ctypes.data)
                out.append(RunRecord(recs, FactorPair(w, h), nx))
    finally:
        for ctx in pool:
            ctx.close()
    return out


def run_csr(offsets, col_idx, vals, m, n, w0, h0, cfg: SolverConfig,
            timing: TimingMode = TimingMode.wall) -> RunRecord:
    """enmf::run<SparseMatrix> on the calling thread's GPU context."""
    return default_context().run_csr(offsets, col_idx, vals, m, n, w0, h0, cfg, timing)


def gram(a):
    return default_context().gram(a)


def cross_wx(w, x):
    return default_context().cross_wx(w, x)


def cross_xht(x, h):
    return default_context().cross_xht(x, h)


def frob_norm_sq(x):
    return default_context().frob_norm_sq(x)


def fast_error(norm_x_sq, w, xht, hht):
    return default_context().fast_error(norm_x_sq, w, xht, hht)


def hals_solve(gram_, cross, h0, max_sweeps, stall_fraction=0.01):
    return default_context().hals_solve(gram_, cross, h0, max_sweeps, stall_fraction)


def optimal_beta_linesearch(x, w_n, w, h_y):
    return default_context().optimal_beta_linesearch(x, w_n, w, h_y)


def active_set_solve(gram_, cross, h0):
    return default_context().active_set_solve(gram_, cross, h0)

"""ctypes front-end to the CPU parity checkers.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_1805_06604_b200) never imports this module.

Two libraries, same signatures:
  * ``Oracle("port")``      -> oracle/liboracle.so, the plain-C restatement
                               (enmf_oracle.c), built by oracle/Makefile.
  * ``Oracle("reference")`` -> oracle/_ref/libenmf_ref.so, the unmodified
                               reference headers compiled in place
                               (ref_shim.cpp); present wherever it was built.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libenmf_ref.so")

ENMF_OK, ENMF_INVALID_ARGUMENT, ENMF_NON_FINITE, ENMF_NO_CONVERGENCE, \
    ENMF_DEGENERATE_COLUMN, ENMF_CUDA_ERROR, ENMF_CACHE_STALE = range(7)


class Config(C.Structure):
    """Mirror of enmf_gpu_config (include/enmf_gpu.h)."""
    _fields_ = [
        ("inner_h", C.c_int32), ("inner_w", C.c_int32), ("hp", C.c_int32),
        ("extrapolation_enabled", C.c_int32),
        ("beta0", C.c_double), ("gamma", C.c_double), ("gamma_bar", C.c_double),
        ("eta", C.c_double), ("max_outer_iterations", C.c_uint64),
        ("max_seconds", C.c_double), ("literal_hp1_order", C.c_int32),
        ("timing", C.c_int32), ("inner_sweep_ratio", C.c_double),
        ("inner_stall_fraction", C.c_double), ("inner_max_sweeps", C.c_uint64),
        ("reinit_seed", C.c_uint64), ("precision", C.c_int32), ("reserved", C.c_int32),
    ]


class Iter(C.Structure):
    """Mirror of enmf_gpu_iter."""
    _fields_ = [
        ("iteration", C.c_uint64), ("elapsed_seconds", C.c_double), ("error", C.c_double),
        ("relative_error", C.c_double), ("beta", C.c_double), ("restarted", C.c_int32),
        ("inner_h_count", C.c_int32), ("inner_w_count", C.c_int32),
        ("reinit_events", C.c_int32),
    ]


class Beta(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("beta", "beta_bar", "beta_prev", "gamma", "gamma_bar", "eta")]


def default_config(**kw) -> Config:
    """enmf::SolverConfig defaults (engine.hpp:149-173)."""
    c = Config(inner_h=0, inner_w=0, hp=1, extrapolation_enabled=1, beta0=0.5, gamma=1.1,
               gamma_bar=1.05, eta=1.5, max_outer_iterations=500, max_seconds=float("inf"),
               literal_hp1_order=0, timing=1, inner_sweep_ratio=0.5, inner_stall_fraction=0.01,
               inner_max_sweeps=0, reinit_seed=0, precision=0, reserved=0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def preset(name: str, **kw) -> Config:
    """enmf::detail::algorithm_config (bench.hpp:108-135), restated."""
    c = default_config()
    if name == "anls":
        c.inner_h = c.inner_w = 0
        c.extrapolation_enabled = 0
    elif name in ("e-anls-hp1", "e-anls-hp3"):
        c.inner_h = c.inner_w = 0
        c.hp = 1 if name == "e-anls-hp1" else 3
        c.beta0, c.gamma, c.gamma_bar, c.eta = 0.5, 1.1, 1.05, 1.5
    elif name == "ahals":
        c.inner_h = c.inner_w = 1
        c.hp = 3
        c.extrapolation_enabled = 0
    elif name in ("e-ahals-hp1", "e-ahals-hp3"):
        c.inner_h = c.inner_w = 1
        c.hp = 1 if name == "e-ahals-hp1" else 3
        c.beta0, c.gamma, c.gamma_bar, c.eta = 0.5, 1.01, 1.005, 1.5
    else:
        raise ValueError(f"unknown algorithm '{name}'")
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def build(quiet: bool = True) -> None:
    """Build liboracle.so (and _ref when /root/reference exists)."""
    subprocess.run(["make", "-C", HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    """One of the two CPU checkers; see module doc."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            if kind == "port" or os.path.isdir("/root/reference/proj/include"):
                build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = L = C.CDLL(path)
        p = "orc_" if kind == "port" else "ref_"
        self.p = p
        run_args = [_dp, _sz, _sz, _dp, _dp, _sz, C.POINTER(Config), C.POINTER(Iter), _sz,
                    C.POINTER(_sz), _dp, _dp, C.POINTER(C.c_double)]
        getattr(L, p + "run_dense").argtypes = run_args
        getattr(L, p + "run_dense").restype = C.c_int
        getattr(L, p + "run_csr").argtypes = [_up, _up, _dp, _sz, _sz, _sz] + run_args[3:]
        getattr(L, p + "run_csr").restype = C.c_int
        getattr(L, p + "last_error").restype = C.c_char_p
        if kind == "port":
            L.orc_gram.argtypes = [_dp, _sz, _sz, _dp]
            L.orc_cross_wx.argtypes = [_dp, _dp, _sz, _sz, _sz, _dp]
            L.orc_cross_xht.argtypes = [_dp, _dp, _sz, _sz, _sz, _dp]
            L.orc_frob_norm_sq.argtypes = [_dp, _sz]
            L.orc_frob_norm_sq.restype = C.c_double
            L.orc_fast_error.argtypes = [C.c_double, _dp, _dp, _dp, _sz, _sz]
            L.orc_fast_error.restype = C.c_double
            L.orc_hals_solve.argtypes = [_dp, _dp, _dp, _sz, _sz, C.c_uint64, C.c_double, _dp,
                                         C.POINTER(C.c_int32)]
            L.orc_active_set_solve.argtypes = [_dp, _dp, _dp, _sz, _sz, _dp, C.POINTER(C.c_int32)]
            L.orc_update_beta.argtypes = [Beta, C.c_int]
            L.orc_update_beta.restype = Beta
            L.orc_gen_lowrank.argtypes = [_sz, _sz, _sz, C.c_uint64, _dp]
            L.orc_gen_fullrank.argtypes = [_sz, _sz, C.c_uint64, _dp]
            L.orc_random_init.argtypes = [_sz, _sz, _sz, C.c_uint64, _dp, _dp]
            L.orc_mix_seed.argtypes = [C.c_uint64] * 3
            L.orc_mix_seed.restype = C.c_uint64
            L.orc_gen_config.argtypes = [C.c_int, _sz, _sz, _sz, C.c_uint64, _dp]
            L.orc_gen_docs.argtypes = [_sz, _sz, C.c_double, C.c_uint64,
                                       C.POINTER(C.POINTER(C.c_uint64)),
                                       C.POINTER(C.POINTER(C.c_uint64)),
                                       C.POINTER(C.POINTER(C.c_double)), C.POINTER(_sz)]
            L.orc_free.argtypes = [C.c_void_p]
            L.orc_derive_max_sweeps.argtypes = [C.c_double, C.c_double, C.c_double]
            L.orc_derive_max_sweeps.restype = C.c_uint64
            L.orc_config_validate.argtypes = [C.POINTER(Config)]
            L.orc_set_threads.argtypes = [C.c_int]
            L.orc_get_threads.restype = C.c_int
            L.orc_gen_tiled.argtypes = [_sz, _sz, _sz, C.c_uint64, _sz, _dp]
        else:
            L.ref_gram.argtypes = [_dp, _sz, _sz, _dp]
            L.ref_cross_wx.argtypes = [_dp, _dp, _sz, _sz, _sz, _dp]
            L.ref_cross_xht.argtypes = [_dp, _dp, _sz, _sz, _sz, _dp]
            L.ref_fast_error.argtypes = [C.c_double, _dp, _dp, _dp, _sz, _sz, C.POINTER(C.c_double)]
            L.ref_hals_solve.argtypes = [_dp, _dp, _dp, _sz, _sz, C.c_uint64, C.c_double, _dp]
            L.ref_active_set_solve.argtypes = [_dp, _dp, _dp, _sz, _sz, _dp]
            L.ref_update_beta.argtypes = [C.POINTER(Beta), C.c_int, C.POINTER(Beta)]
            L.ref_gen_lowrank.argtypes = [_sz, _sz, _sz, C.c_uint64, _dp]
            L.ref_random_init.argtypes = [_sz, _sz, _sz, C.c_uint64, _dp, _dp]
            L.ref_mix_seed.argtypes = [C.c_uint64] * 3
            L.ref_mix_seed.restype = C.c_uint64

    def _check(self, rc):
        if rc != ENMF_OK:
            raise OracleError(rc, getattr(self.lib, self.p + "last_error")().decode())

    # ---- run -------------------------------------------------------------
    def run_dense(self, x, w0, h0, cfg: Config):
        x, w0, h0 = _c(x), _c(w0), _c(h0)
        m, n = x.shape
        r = w0.shape[1]
        cap = int(cfg.max_outer_iterations) + 1
        iters = (Iter * cap)()
        nit = _sz(0)
        w = np.zeros((m, r))
        h = np.zeros((r, n))
        nx = C.c_double(0)
        rc = getattr(self.lib, self.p + "run_dense")(x, m, n, w0, h0, r, C.byref(cfg), iters, cap,
                                                     C.byref(nit), w, h, C.byref(nx))
        self._check(rc)
        return records(iters, nit.value), w, h, nx.value

    def run_csr(self, off, cidx, vals, m, n, w0, h0, cfg: Config):
        off, cidx, vals, w0, h0 = _c(off, np.uint64), _c(cidx, np.uint64), _c(vals), _c(w0), _c(h0)
        r = w0.shape[1]
        cap = int(cfg.max_outer_iterations) + 1
        iters = (Iter * cap)()
        nit = _sz(0)
        w = np.zeros((m, r))
        h = np.zeros((r, n))
        nx = C.c_double(0)
        rc = getattr(self.lib, self.p + "run_csr")(off, cidx, vals, m, n, len(vals), w0, h0, r,
                                                   C.byref(cfg), iters, cap, C.byref(nit), w, h,
                                                   C.byref(nx))
        self._check(rc)
        return records(iters, nit.value), w, h, nx.value

    # ---- kernels ---------------------------------------------------------
    def gram(self, a):
        a = _c(a)
        g = np.zeros((a.shape[1], a.shape[1]))
        getattr(self.lib, self.p + "gram")(a, a.shape[0], a.shape[1], g)
        return g

    def cross_wx(self, w, x):
        w, x = _c(w), _c(x)
        out = np.zeros((w.shape[1], x.shape[1]))
        getattr(self.lib, self.p + "cross_wx")(w, x, x.shape[0], x.shape[1], w.shape[1], out)
        return out

    def cross_xht(self, x, h):
        x, h = _c(x), _c(h)
        out = np.zeros((x.shape[0], h.shape[0]))
        getattr(self.lib, self.p + "cross_xht")(x, h, x.shape[0], x.shape[1], h.shape[0], out)
        return out

    def fast_error(self, nx2, w, xht, hht):
        w, xht, hht = _c(w), _c(xht), _c(hht)
        if self.kind == "port":
            return self.lib.orc_fast_error(nx2, w, xht, hht, w.shape[0], w.shape[1])
        e = C.c_double()
        self._check(self.lib.ref_fast_error(nx2, w, xht, hht, w.shape[0], w.shape[1], C.byref(e)))
        return e.value

    def hals_solve(self, gram, cross, h0, max_sweeps, stall=0.01):
        gram, cross, h0 = _c(gram), _c(cross), _c(h0)
        h = np.zeros_like(h0)
        r, n = h0.shape
        if self.kind == "port":
            sw = C.c_int32()
            self._check(self.lib.orc_hals_solve(gram, cross, h0, r, n, max_sweeps, stall, h, C.byref(sw)))
            return h, sw.value
        self._check(self.lib.ref_hals_solve(gram, cross, h0, r, n, max_sweeps, stall, h))
        return h, None

    def active_set_solve(self, gram, cross, h0):
        gram, cross, h0 = _c(gram), _c(cross), _c(h0)
        h = np.zeros_like(h0)
        r, n = h0.shape
        if self.kind == "port":
            rd = C.c_int32()
            self._check(self.lib.orc_active_set_solve(gram, cross, h0, r, n, h, C.byref(rd)))
            return h, rd.value
        self._check(self.lib.ref_active_set_solve(gram, cross, h0, r, n, h))
        return h, None

    def update_beta(self, s: dict, dec: bool) -> dict:
        b = Beta(**s)
        if self.kind == "port":
            o = self.lib.orc_update_beta(b, int(dec))
        else:
            o = Beta()
            self.lib.ref_update_beta(C.byref(b), int(dec), C.byref(o))
        return {k: getattr(o, k) for k, _ in Beta._fields_}

    # ---- data ------------------------------------------------------------
    def gen_lowrank(self, m, n, r, seed):
        x = np.zeros((m, n))
        getattr(self.lib, self.p + "gen_lowrank")(m, n, r, seed, x)
        return x

    def random_init(self, m, n, r, seed):
        w = np.zeros((m, r))
        h = np.zeros((r, n))
        getattr(self.lib, self.p + "random_init")(m, n, r, seed, w, h)
        return w, h

    def mix_seed(self, b, x=0, y=0):
        return getattr(self.lib, self.p + "mix_seed")(b, x, y)

    def gen_config(self, which, m, n, r, seed):
        x = np.zeros((m, n))
        self._check(self.lib.orc_gen_config(which, m, n, r, seed, x))
        return x

    def gen_tiled(self, m, n, r, seed, tile=4096, threads=None):
        """C5 data on tiles with per-tile streams (replica.c orc_gen_tiled); any thread count
        gives the same bits."""
        x = np.empty((m, n))
        old = self.threads
        self.threads = threads or os.cpu_count() or 1
        try:
            self._check(self.lib.orc_gen_tiled(m, n, r, seed, tile, x))
        finally:
            self.threads = old
        return x

    @property
    def threads(self) -> int:
        """Replica threads for run_dense / time_steps (1 = the plain single-threaded port)."""
        return self.lib.orc_get_threads()

    @threads.setter
    def threads(self, n: int) -> None:
        self.lib.orc_set_threads(int(n))

    def gen_docs(self, m, n, seed, zipf_s=1.1):
        po, pc, pv = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)(), C.POINTER(C.c_double)()
        nnz = _sz()
        self._check(self.lib.orc_gen_docs(m, n, zipf_s, seed, C.byref(po), C.byref(pc),
                                          C.byref(pv), C.byref(nnz)))
        k = nnz.value
        off = np.ctypeslib.as_array(po, shape=(m + 1,)).copy()
        cidx = np.ctypeslib.as_array(pc, shape=(k,)).copy() if k else np.zeros(0, np.uint64)
        vals = np.ctypeslib.as_array(pv, shape=(k,)).copy() if k else np.zeros(0)
        for p in (po, pc, pv):
            self.lib.orc_free(C.cast(p, C.c_void_p))
        return off, cidx, vals


def records(iters, count):
    """enmf_gpu_iter array -> dict of numpy arrays (one entry per record)."""
    k = min(count, len(iters))
    return {
        "iteration": np.array([iters[i].iteration for i in range(k)], dtype=np.int64),
        "error": np.array([iters[i].error for i in range(k)]),
        "relative_error": np.array([iters[i].relative_error for i in range(k)]),
        "beta": np.array([iters[i].beta for i in range(k)]),
        "restarted": np.array([iters[i].restarted for i in range(k)], dtype=np.int32),
        "inner_h": np.array([iters[i].inner_h_count for i in range(k)], dtype=np.int32),
        "inner_w": np.array([iters[i].inner_w_count for i in range(k)], dtype=np.int32),
        "reinit": np.array([iters[i].reinit_events for i in range(k)], dtype=np.int32),
        "elapsed": np.array([iters[i].elapsed_seconds for i in range(k)]),
    }

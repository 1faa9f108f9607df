"""ctypes binding of libenmf_gpu.so (include/enmf_gpu.h).

The shared library is built in-tree (csrc/Makefile, __graft_entry__.build()).
There is no CPU fallback: if the library or a CUDA device is missing, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ENMF_GPU_LIB") or os.path.join(HERE, "libenmf_gpu.so")   # override: A/B timing of builds

ENMF_OK = 0
ENMF_INVALID_ARGUMENT = 1
ENMF_NON_FINITE = 2
ENMF_NO_CONVERGENCE = 3
ENMF_DEGENERATE_COLUMN = 4
ENMF_CUDA_ERROR = 5
ENMF_CACHE_STALE = 6
ENMF_PARSE_ERROR = 7
ENMF_UNSUPPORTED_FORMAT = 8
ENMF_IO_ERROR = 9
ENMF_ZERO_DIRECTION = 10

ENMF_INNER_EXACT, ENMF_INNER_HALS = 0, 1
ENMF_TIMING_WALL, ENMF_TIMING_NONE = 0, 1
ENMF_PRECISION_FP64, ENMF_PRECISION_TF32, ENMF_PRECISION_FP64_EXACT = 0, 1, 2


class CConfig(C.Structure):
    """enmf_gpu_config — 1:1 with enmf::SolverConfig (engine.hpp:149-173)."""
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


class CIter(C.Structure):
    """enmf_gpu_iter — enmf::IterationRecord (engine.hpp:216-223) + instrumentation."""
    _fields_ = [
        ("iteration", C.c_uint64), ("elapsed_seconds", C.c_double), ("error", C.c_double),
        ("relative_error", C.c_double), ("beta", C.c_double), ("restarted", C.c_int32),
        ("inner_h_count", C.c_int32), ("inner_w_count", C.c_int32),
        ("reinit_events", C.c_int32),
    ]


class CBeta(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("beta", "beta_bar", "beta_prev", "gamma", "gamma_bar", "eta")]


#: every symbol include/enmf_gpu.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "enmf_gpu_config_default", "enmf_gpu_config_preset", "enmf_gpu_config_validate",
    "enmf_gpu_update_beta", "enmf_gpu_create", "enmf_gpu_destroy", "enmf_gpu_last_error",
    "enmf_gpu_kernel_launches", "enmf_gpu_run_dense", "enmf_gpu_run_csr", "enmf_gpu_load_dense",
    "enmf_gpu_solve", "enmf_gpu_set_precision", "enmf_gpu_gram", "enmf_gpu_cross_wx",
    "enmf_gpu_cross_xht", "enmf_gpu_frob_norm_sq", "enmf_gpu_fast_error", "enmf_gpu_hals_solve",
    "enmf_gpu_active_set_solve", "enmf_gpu_begin", "enmf_gpu_step", "enmf_gpu_step_profiled",
    "enmf_gpu_sync", "enmf_gpu_end", "enmf_gpu_stream", "enmf_gpu_digit_levels",
    "enmf_gpu_dist_shard", "enmf_gpu_dist_alloc", "enmf_gpu_dist_init", "enmf_gpu_load_dense_sharded",
    "enmf_gpu_dist_finalize", "enmf_gpu_dist_selftest", "enmf_gpu_hals_solve_vranks", "enmf_gpu_load_csr", "enmf_gpu_last_error_line",
    "enmf_gpu_optimal_beta_linesearch", "enmf_gpu_optimal_beta_linesearch_csr",
    "enmf_gpu_batch_eligible", "enmf_gpu_run_batch_dense",
    # data formats and generators (csrc/io.cpp)
    "enmf_io_read_matrix_market", "enmf_io_read_dense_csv", "enmf_io_matrix_shape",
    "enmf_io_matrix_offsets", "enmf_io_matrix_col_indices", "enmf_io_matrix_values",
    "enmf_io_matrix_free", "enmf_io_write_matrix_market", "enmf_io_write_dense_csv",
    "enmf_io_write_run_csv", "enmf_io_format_double", "enmf_mix_seed", "enmf_uniform_matrix",
    "enmf_random_init", "enmf_lowrank_factors", "enmf_gen_lowrank", "enmf_gen_fullrank", "enmf_gen_tiled",
]

#: entry points that do not return an ENMF_* status
_NON_STATUS = ("enmf_gpu_config_default", "enmf_gpu_destroy", "enmf_gpu_last_error",
               "enmf_gpu_kernel_launches", "enmf_gpu_update_beta", "enmf_gpu_stream",
               "enmf_gpu_dist_shard", "enmf_gpu_last_error_line", "enmf_io_matrix_shape",
               "enmf_io_matrix_offsets", "enmf_io_matrix_col_indices", "enmf_io_matrix_values",
               "enmf_io_matrix_free", "enmf_io_format_double", "enmf_mix_seed")

_lib = None


def load() -> C.CDLL:
    """Load libenmf_gpu.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    sz, dp, vp = C.c_size_t, C.c_void_p, C.c_void_p
    ip = C.POINTER(C.c_int32)
    L.enmf_gpu_config_default.argtypes = [C.POINTER(CConfig)]
    L.enmf_gpu_config_default.restype = None
    L.enmf_gpu_config_preset.argtypes = [C.POINTER(CConfig), C.c_char_p]
    L.enmf_gpu_config_validate.argtypes = [C.POINTER(CConfig)]
    L.enmf_gpu_update_beta.argtypes = [CBeta, C.c_int]
    L.enmf_gpu_update_beta.restype = CBeta
    L.enmf_gpu_create.argtypes = [C.POINTER(vp), C.c_int]
    L.enmf_gpu_destroy.argtypes = [vp]
    L.enmf_gpu_destroy.restype = None
    L.enmf_gpu_last_error.restype = C.c_char_p
    L.enmf_gpu_kernel_launches.argtypes = [vp]
    L.enmf_gpu_kernel_launches.restype = C.c_uint64
    run_tail = [sz, C.POINTER(CConfig), C.POINTER(CIter), sz, C.POINTER(sz), dp, dp, C.POINTER(C.c_double)]
    L.enmf_gpu_run_dense.argtypes = [vp, dp, sz, sz, dp, dp] + run_tail
    L.enmf_gpu_run_csr.argtypes = [vp, dp, dp, dp, sz, sz, sz, dp, dp] + run_tail
    L.enmf_gpu_load_dense.argtypes = [vp, dp, sz, sz, C.c_int]
    L.enmf_gpu_batch_eligible.argtypes = [sz, sz, sz, C.POINTER(CConfig)]
    L.enmf_gpu_run_batch_dense.argtypes = [vp, sz, dp, sz, sz, dp, dp, sz, C.POINTER(CConfig), C.POINTER(CIter), sz,
                                           ip, ip, dp, dp, dp]
    L.enmf_gpu_load_csr.argtypes = [vp, dp, dp, dp, sz, sz, sz]
    L.enmf_gpu_solve.argtypes = [vp, dp, dp, sz, C.c_int, C.POINTER(CConfig), C.POINTER(CIter), sz,
                                 C.POINTER(sz), dp, dp, C.POINTER(C.c_double)]
    L.enmf_gpu_set_precision.argtypes = [vp, C.c_int]
    L.enmf_gpu_gram.argtypes = [vp, dp, sz, sz, dp]
    L.enmf_gpu_cross_wx.argtypes = [vp, dp, dp, sz, sz, sz, dp]
    L.enmf_gpu_cross_xht.argtypes = [vp, dp, dp, sz, sz, sz, dp]
    L.enmf_gpu_frob_norm_sq.argtypes = [vp, dp, sz, C.POINTER(C.c_double)]
    L.enmf_gpu_fast_error.argtypes = [vp, C.c_double, dp, dp, dp, sz, sz, C.POINTER(C.c_double)]
    L.enmf_gpu_hals_solve.argtypes = [vp, dp, dp, dp, sz, sz, C.c_uint64, C.c_double, dp, ip]
    L.enmf_gpu_active_set_solve.argtypes = [vp, dp, dp, dp, sz, sz, dp, ip]
    L.enmf_gpu_begin.argtypes = [vp, dp, dp, sz, C.c_int, C.POINTER(CConfig)]
    L.enmf_gpu_step.argtypes = [vp, C.c_uint64]
    L.enmf_gpu_step_profiled.argtypes = [vp, C.POINTER(C.c_double), sz]
    L.enmf_gpu_sync.argtypes = [vp, C.POINTER(CIter), sz, C.POINTER(sz)]
    L.enmf_gpu_end.argtypes = [vp, dp, dp, C.POINTER(C.c_double)]
    L.enmf_gpu_stream.argtypes = [vp]
    L.enmf_gpu_stream.restype = C.c_void_p
    szp = C.POINTER(sz)
    L.enmf_gpu_dist_shard.argtypes = [sz, sz, C.c_int, C.c_int, szp, szp, szp, szp]
    L.enmf_gpu_dist_shard.restype = None
    L.enmf_gpu_dist_alloc.argtypes = [vp, C.c_int, C.c_int, sz, sz, sz, C.c_void_p]
    L.enmf_gpu_dist_init.argtypes = [vp, C.c_void_p]
    L.enmf_gpu_load_dense_sharded.argtypes = [vp, dp, dp, C.c_int]
    L.enmf_gpu_dist_finalize.argtypes = [vp]
    L.enmf_gpu_hals_solve_vranks.argtypes = [vp, C.c_void_p, C.c_void_p, C.c_void_p, sz, sz, C.c_int, C.c_uint64,
                                             C.c_double, C.c_void_p, C.c_void_p]
    L.enmf_gpu_dist_selftest.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, sz, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
    L.enmf_gpu_last_error_line.restype = sz
    L.enmf_gpu_optimal_beta_linesearch.argtypes = [vp, dp, sz, sz, dp, dp, dp, sz, C.POINTER(C.c_double)]
    L.enmf_gpu_optimal_beta_linesearch_csr.argtypes = [vp, dp, dp, dp, sz, sz, sz, dp, dp, dp, sz,
                                                       C.POINTER(C.c_double)]
    u64p = C.POINTER(C.c_uint64)
    L.enmf_io_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.enmf_io_read_dense_csv.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.enmf_io_matrix_shape.argtypes = [vp, szp, szp, szp, ip]
    L.enmf_io_matrix_shape.restype = None
    L.enmf_io_matrix_offsets.argtypes = [vp]
    L.enmf_io_matrix_offsets.restype = u64p
    L.enmf_io_matrix_col_indices.argtypes = [vp]
    L.enmf_io_matrix_col_indices.restype = u64p
    L.enmf_io_matrix_values.argtypes = [vp]
    L.enmf_io_matrix_values.restype = C.POINTER(C.c_double)
    L.enmf_io_matrix_free.argtypes = [vp]
    L.enmf_io_matrix_free.restype = None
    L.enmf_io_write_matrix_market.argtypes = [C.c_char_p, dp, dp, dp, sz, sz]
    L.enmf_io_write_dense_csv.argtypes = [C.c_char_p, dp, sz, sz]
    L.enmf_io_write_run_csv.argtypes = [C.c_char_p, C.POINTER(CIter), sz, C.c_double]
    L.enmf_io_format_double.argtypes = [C.c_double, C.c_char_p, sz]
    L.enmf_io_format_double.restype = sz
    L.enmf_mix_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    L.enmf_mix_seed.restype = C.c_uint64
    L.enmf_uniform_matrix.argtypes = [sz, sz, C.c_uint64, dp]
    L.enmf_random_init.argtypes = [sz, sz, sz, C.c_uint64, dp, dp]
    L.enmf_lowrank_factors.argtypes = [sz, sz, sz, C.c_uint64, dp, dp]
    L.enmf_gen_lowrank.argtypes = [sz, sz, sz, C.c_uint64, dp]
    L.enmf_gen_tiled.argtypes = [sz, sz, sz, C.c_uint64, sz, sz, sz, sz, sz, dp]
    L.enmf_gen_fullrank.argtypes = [sz, sz, C.c_uint64, dp]
    for name in EXPORTS:
        fn = getattr(L, name)
        if name not in _NON_STATUS:
            fn.restype = C.c_int
    _lib = L
    return L

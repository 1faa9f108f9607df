"""B200-native hot path of extrapolated NMF (E-A-HALS / E-ANLS, arXiv 1805.06604).

A drop-in for enmf::run / enmf::step of the reference C++ library: the same
SolverConfig, W/H layouts and error behaviour, computed by hand-written sm_100a
CUDA kernels (libenmf_gpu.so, C-ABI in include/enmf_gpu.h).  See DESIGN.md.
"""
from .enmf import (  # noqa: F401
    BetaSchedule, CacheStale, Context, DEFAULT_ALGORITHMS, DegenerateColumn, DeviceError, FactorPair,
    InnerSolver, InvalidArgument, IterationRecord, NoConvergence, NonFiniteIterate, Precision, RunRecord,
    SolverConfig, TimingMode, active_set_solve, algorithm_config, cross_wx, cross_xht, default_context,
    fast_error, frob_norm_sq, gram, hals_solve, run, run_batch, run_csr, update_beta,
)
from ._lib import LIB_PATH, load as load_library  # noqa: F401

"""B200-native hot path of extrapolated NMF (E-A-HALS / E-ANLS, arXiv 1805.06604).

A drop-in for enmf::run / enmf::step of the reference C++ library: the same
SolverConfig, W/H layouts and error behaviour, computed by hand-written sm_100a
CUDA kernels (libenmf_gpu.so, C-ABI in include/enmf_gpu.h).  See DESIGN.md.
"""
from .enmf import (  # noqa: F401
    BetaSchedule, CacheStale, Context, DEFAULT_ALGORITHMS, DegenerateColumn, DeviceError, FactorPair,
    InnerSolver, InvalidArgument, IterationRecord, NoConvergence, NonFiniteIterate, Precision, RunRecord,
    SolverConfig, TimingMode, active_set_solve, algorithm_config, cross_wx, cross_xht, default_context,
    fast_error, frob_norm_sq, gram, hals_solve, IoError, optimal_beta_linesearch, ZeroDirection, ParseError, run, run_batch, run_batch_packed, batch_eligible, run_csr, UnsupportedFormat,
    update_beta,
)
from . import data, suite  # noqa: F401  (enmf/data.hpp formats + generators; enmf/bench.hpp suites)
from .data import (  # noqa: F401
    SparseMatrix, format_double, gen_fullrank, gen_lowrank, lowrank_factors, mix_seed, random_init,
    read_dense_csv, read_matrix_market, uniform_matrix, write_dense_csv, write_matrix_market, write_run_csv,
)
from .suite import (  # noqa: F401
    AlgorithmSpec, Budget, DatasetKind, DatasetSpec, SuiteResults, SuiteSpec, compute_curves,
    compute_curves_for_dataset, emit, load_dataset, make_algorithm, rank_final_errors, run_suite,
)
from ._lib import LIB_PATH, load as load_library  # noqa: F401

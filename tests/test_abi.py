"""CPU tier: the C-ABI library loads and exports every symbol include/enmf_gpu.h
declares; host-side logic (presets, validation, update_beta) without a GPU."""
import ctypes as C
import os
import re

import pytest

import paper_1805_06604_b200 as E
from paper_1805_06604_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "enmf_gpu.h")).read()
    return sorted(set(re.findall(r"\b(enmf_(?:gpu|io|mix|uniform|random|lowrank|gen)_?\w*)\s*\(", src)))


def test_library_exports_header():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_presets_match_reference_table():
    """bench.hpp:108-135."""
    c = E.algorithm_config("e-ahals-hp3")
    assert (c.inner_h, c.inner_w, c.hp, c.beta0, c.gamma, c.gamma_bar, c.eta) == \
        (E.InnerSolver.hals, E.InnerSolver.hals, 3, 0.5, 1.01, 1.005, 1.5)
    c = E.algorithm_config("e-anls-hp1")
    assert (c.inner_h, c.hp, c.gamma, c.gamma_bar) == (E.InnerSolver.exact, 1, 1.1, 1.05)
    assert not E.algorithm_config("anls").extrapolation_enabled
    assert not E.algorithm_config("ahals").extrapolation_enabled
    with pytest.raises(E.InvalidArgument):
        E.algorithm_config("nope")


def test_config_validation_host():
    E.SolverConfig().validate()
    for kw in [dict(hp=0), dict(beta0=1.0), dict(gamma=1.01, gamma_bar=1.02), dict(max_seconds=0.0),
               dict(inner_sweep_ratio=0.0), dict(inner_stall_fraction=0.0)]:
        with pytest.raises(E.InvalidArgument):
            E.SolverConfig(**kw).validate()
    # beta0 = 0 skips the schedule check (engine.hpp:180)
    E.SolverConfig(beta0=0.0, gamma=1.0, gamma_bar=1.0).validate()


def test_update_beta_matches_oracle(port):
    import numpy as np
    rng = np.random.default_rng(1)
    for _ in range(500):
        s = dict(beta=float(rng.random()), beta_bar=float(rng.random()), beta_prev=float(rng.random()),
                 gamma=1.1, gamma_bar=1.05, eta=1.5)
        d = bool(rng.integers(2))
        a = E.update_beta(E.BetaSchedule(**s), d)
        b = port.update_beta(s, d)
        assert a.__dict__ == b


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(E.DeviceError):
        E.Context()

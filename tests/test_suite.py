"""The experiment harness (suite.py ≙ bench.hpp): specs, datasets, curves, ranking, emit,
and run_suite on the GPU.

Pinned against tests/golden/suite/emit/ — the reference's own run_suite + emit() output
for tests/golden/suite/spec.json (4 datasets incl. a Matrix Market and a CSV file,
2 inits, all 6 algorithms, 30 iterations; tests/golden/make_golden_io.py):
  * CPU: the run traces are read back into SuiteResults and emit() must reproduce the
    reference's curve CSVs and summary.json byte for byte (curves, floors, ranking and
    the JSON layout are pure host logic);
  * GPU: run_suite itself with precision=fp64_exact must reproduce every one of the 73
    files byte for byte; the fp64 product path must match every trace within 1e-9
    relative error (or the trace identity's own cancellation bound below it) with
    identical restarts.
"""
import csv
import json
import math
import os

import numpy as np
import pytest

from paper_1805_06604_b200 import data as D
from paper_1805_06604_b200 import enmf as E
from paper_1805_06604_b200 import suite as S

GOLD = os.path.join(os.path.dirname(__file__), "golden", "suite")
SPEC = json.load(open(os.path.join(GOLD, "spec.json")))


def make_spec(precision=E.Precision.fp64, threads=None):
    ds = [S.DatasetSpec(kind=S.DatasetKind(d["kind"]), m=d.get("m", 0), n=d.get("n", 0), r=d["r"],
                        seed=d.get("seed", 0), path=d.get("path", ""), name=d.get("name", ""))
          for d in SPEC["datasets"]]
    return S.SuiteSpec(datasets=ds, algorithms=[S.make_algorithm(a) for a in SPEC["algorithms"]],
                       inits_per_dataset=SPEC["inits_per_dataset"],
                       budget=S.Budget(max_iterations=SPEC["max_iterations"]), base_seed=SPEC["base_seed"],
                       threads=SPEC["threads"] if threads is None else threads, wall_timing=SPEC["wall_timing"],
                       precision=precision)


def run_file(spec, r):
    return os.path.join(GOLD, "emit", f"run_{S.dataset_label(spec.datasets[r.dataset_index], r.dataset_index)}_"
                                      f"{S.sanitize_label(spec.algorithms[r.algorithm_index].name)}_{r.init_index}.csv")


def results_from_traces(spec):
    """SuiteResults whose records are the reference's traces (rel_err, beta, restarted)."""
    nd, ni, na = len(spec.datasets), spec.inits_per_dataset, len(spec.algorithms)
    res = S.SuiteResults(spec=spec)
    for t in range(nd * ni * na):
        r = S.RunResult(t // (na * ni), (t // na) % ni, t % na)
        with open(run_file(spec, r)) as f:
            rows = list(csv.DictReader(f))
        r.record = E.RunRecord([E.IterationRecord(int(x["iter"]), float(x["elapsed_s"]), 0.0, float(x["rel_err"]),
                                                  float(x["beta"]), x["restarted"] == "1") for x in rows])
        res.runs.append(r)
    return res


def test_emit_reproduces_reference_artifacts_from_traces(tmp_path):
    spec = make_spec()
    res = results_from_traces(spec)
    written = S.emit(res, tmp_path / "out")
    names = sorted(os.listdir(os.path.join(GOLD, "emit")))
    assert sorted(os.path.basename(p) for p in written) == names
    for p in written:
        want = open(os.path.join(GOLD, "emit", os.path.basename(p)), "rb").read()
        assert open(p, "rb").read() == want, os.path.basename(p)


def test_curves_and_ranking_semantics():
    """test_bench.cpp:218-310: floors, padding of short runs, MixedDatasets, MissingRun."""
    spec = make_spec()
    res = results_from_traces(spec)
    zero = S.compute_curves_for_dataset(res, 0)          # lowrank: floor 0
    assert zero.e_min == 0.0 and len(zero.per_algorithm) == 6
    best = S.compute_curves_for_dataset(res, 1)          # fullrank: shared best floor
    finals = [r.record.final_relative_error() for r in res.runs if r.dataset_index == 1]
    assert best.e_min == min(finals)
    assert min(rc.points[-1].e for rc in best.per_run) == 0.0
    with pytest.raises(S.MixedDatasets):
        S.compute_curves(res.runs, S.EminPolicy.shared_best)
    # a short run is padded with its final point
    short = S.RunResult(0, 0, 0, E.RunRecord([E.IterationRecord(0, 0.0, 0, 0.5, 0.5, False),
                                              E.IterationRecord(1, 0.0, 0, 0.25, 0.5, False)]))
    longr = S.RunResult(0, 1, 0, E.RunRecord([E.IterationRecord(k, 0.0, 0, 1.0 / (k + 1), 0.5, False)
                                              for k in range(4)]))
    cs = S.compute_curves([short, longr], S.EminPolicy.zero)
    assert [p.e for p in cs.per_algorithm[0].points] == [(0.5 + 1.0) / 2, (0.25 + 0.5) / 2,
                                                         (0.25 + 1 / 3) / 2, (0.25 + 0.25) / 2]
    table = S.rank_final_errors(res)
    assert table.group_count == 4 * 2
    for pos in range(6):
        assert sum(row.ranking[pos] for row in table.rows) == table.group_count
    res.runs[3].failed, res.runs[3].failure = True, "synthetic failure"
    with pytest.raises(S.MissingRun):
        S.rank_final_errors(res)


def test_specs_labels_and_dataset_loading(tmp_path):
    """test_bench.cpp:104-152."""
    d = S.DatasetSpec(S.DatasetKind.lowrank, 10, 8, 3, 1)
    d.validate()
    for bad in (S.DatasetSpec(S.DatasetKind.lowrank, 10, 8, 9, 1), S.DatasetSpec(S.DatasetKind.lowrank, 10, 8, 0, 1),
                S.DatasetSpec(S.DatasetKind.file, r=2)):
        with pytest.raises(E.InvalidArgument):
            bad.validate()
    S.DatasetSpec(S.DatasetKind.file, r=2, path="x.mtx").validate()
    assert S.dataset_label(S.DatasetSpec(S.DatasetKind.lowrank, 4, 4, 2, 0), 3) == "lowrank3"
    assert S.dataset_label(S.DatasetSpec(S.DatasetKind.lowrank, 4, 4, 2, 0, name="my data/set!"), 0) == "my-data-set-"
    rng = np.random.default_rng(161)
    dense = rng.uniform(0, 1, (6, 5))
    D.write_dense_csv(tmp_path / "d.csv", dense)
    sp = D.SparseMatrix.from_triplets(4, 4, [(0, 0, 1.0), (1, 2, 2.0), (3, 3, 3.0)])
    D.write_matrix_market(tmp_path / "s.mtx", sp)
    f = S.DatasetSpec(S.DatasetKind.file, r=2, path=str(tmp_path / "d.csv"))
    assert np.array_equal(S.load_dataset(f), dense)
    f.path = str(tmp_path / "s.mtx")
    assert np.array_equal(S.load_dataset(f).to_dense(), sp.to_dense())
    f.r = 5
    with pytest.raises(E.InvalidArgument):
        S.load_dataset(f)
    f.r, f.path = 2, str(tmp_path / "d.unknown")
    with pytest.raises(E.UnsupportedFormat):
        S.load_dataset(f)
    with pytest.raises(E.IoError):     # load-time errors are raised (test_bench.cpp:208-216)
        S.run_suite(S.SuiteSpec(datasets=[S.DatasetSpec(S.DatasetKind.file, r=2, path="definitely-missing.mtx")],
                                algorithms=[S.make_algorithm("anls")]))
    assert S.default_algorithms() == ["anls", "e-anls-hp1", "e-anls-hp3", "ahals", "e-ahals-hp1", "e-ahals-hp3"]


def test_json_number_layout():
    assert S._json_number(0.5) == "0.5" and S._json_number(13.0) == "13.0"
    assert S._json_number(1e-5) == "1e-05" and S._json_number(0.0001) == "0.0001"
    assert S._json_number(1e15) == "1e+15" and S._json_number(-2.5e-7) == "-2.5e-07"
    assert S._json_number(math.inf) == "null"


# ---------------------------------------------------------------------- GPU
def _run_in_gold_dir(spec):
    cwd = os.getcwd()
    os.chdir(GOLD)            # the spec names its files relative to the suite directory
    try:
        return S.run_suite(spec)
    finally:
        os.chdir(cwd)


@pytest.mark.gpu
def test_run_suite_exact_reproduces_reference_files(tmp_path):
    spec = make_spec(E.Precision.fp64_exact)
    res = _run_in_gold_dir(spec)
    assert res.failed_count() == 0, [r.failure for r in res.runs if r.failed]
    written = S.emit(res, tmp_path / "out")
    assert len(written) == len(os.listdir(os.path.join(GOLD, "emit")))
    for p in written:
        want = open(os.path.join(GOLD, "emit", os.path.basename(p)), "rb").read()
        assert open(p, "rb").read() == want, os.path.basename(p)


@pytest.mark.gpu
def test_run_suite_fp64_matches_reference_traces():
    """The product path (INT8-digit / DMMA products, FMA sweeps) against the reference's
    traces, with the bar the other parity tests use (test_gpu_parity.assert_parity):
    max(1e-9, eps·κ_k) relative, κ_k = 1/rel_err_k², the trace identity's own cancellation
    bound; restarts identical while the reference is above the 1e-6 noise floor (the
    noise-free low-rank dataset reaches it, test_engine.cpp:67-81)."""
    spec = make_spec(E.Precision.fp64)
    res = _run_in_gold_dir(spec)
    assert res.failed_count() == 0
    ref = results_from_traces(spec)
    eps = np.finfo(float).eps
    for got, want in zip(res.runs, ref.runs):
        g = got.record.column("relative_error")
        w = want.record.column("relative_error")
        assert len(g) == len(w)
        below = np.nonzero(w <= 1e-6)[0]
        k = int(below[0]) if len(below) else len(w)
        np.testing.assert_array_equal(got.record.column("restarted")[:k], want.record.column("restarted")[:k])
        dev = np.abs(g[:k] - w[:k]) / w[:k]
        assert np.all(dev <= np.maximum(1e-9, eps / w[:k] ** 2)), (got.dataset_index, got.algorithm_index, dev.max())


@pytest.mark.gpu
def test_run_suite_does_not_depend_on_width():
    """test_bench.cpp:184-206: reruns and different concurrency are bitwise identical."""
    a = _run_in_gold_dir(make_spec(E.Precision.fp64, threads=1))
    b = _run_in_gold_dir(make_spec(E.Precision.fp64, threads=16))
    for x, y in zip(a.runs, b.runs):
        np.testing.assert_array_equal(x.record.column("error"), y.record.column("error"))
        np.testing.assert_array_equal(x.record.factors.w, y.record.factors.w)

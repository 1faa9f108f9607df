"""The paper's experiment protocol on the GPU — the reference's enmf/bench.hpp.

A suite is a grid of (dataset, initialization, algorithm) runs with one initial factor
pair per (dataset, initialization), shared by every algorithm, followed by error
curves, a final-error ranking and CSV/JSON artifacts:

    DatasetSpec / SuiteSpec / Budget / AlgorithmSpec     bench.hpp:54-186
    load_dataset                                        bench.hpp:207-231
    run_suite                                           bench.hpp:233-294
    compute_curves / compute_curves_for_dataset         bench.hpp:296-425
    rank_final_errors                                   bench.hpp:427-480
    dataset_error_floors / emit                         bench.hpp:482-646

run_suite is the batched many-small-runs backend: where the
reference hands each run to a host thread, here `threads` device contexts (each a
CUDA stream with its own per-iteration CUDA graph) take one run each; every run of
a wave is enqueued before any result is read, so the launch-bound small runs overlap
on the GPU.  Each run is computed exactly as `enmf_gpu_run_dense/csr` computes it
alone, so results do not depend on `threads` (bench.hpp:184-206's guarantee); with
`precision=Precision.fp64_exact` they are bitwise the reference's, and so are the
emitted files (tests/test_suite.py checks them byte for byte against the reference's
own emit()).
"""
from __future__ import annotations

import enum
import json
import math
import os
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Union

import numpy as np

from . import data as io
from .enmf import (batch_eligible, run_batch_packed, Context, FactorPair, InvalidArgument, Precision, RunRecord, SolverConfig, TimingMode,
                   UnsupportedFormat, algorithm_config)

__all__ = [
    "DatasetKind", "DatasetSpec", "AlgorithmSpec", "Budget", "SuiteSpec", "RunResult", "SuiteResults",
    "MixedDatasets", "MissingRun", "EminPolicy", "CurvePoint", "RunCurve", "AlgorithmCurve", "CurveSet",
    "RankingRow", "RankingTable", "EmitOptions", "sanitize_label", "dataset_label", "make_algorithm",
    "default_algorithms", "load_dataset", "run_suite", "compute_curves", "compute_curves_for_dataset",
    "rank_final_errors", "dataset_error_floors", "emit",
]


class MixedDatasets(Exception):
    """enmf::MixedDatasets (bench.hpp:42-45, a std::logic_error)."""


class MissingRun(RuntimeError):
    """enmf::MissingRun (bench.hpp:47-50)."""


class DatasetKind(str, enum.Enum):
    lowrank = "lowrank"
    fullrank = "fullrank"
    file = "file"


@dataclass
class DatasetSpec:
    """enmf::DatasetSpec (bench.hpp:63-85)."""
    kind: DatasetKind = DatasetKind.lowrank
    m: int = 0
    n: int = 0
    r: int = 0
    seed: int = 0
    path: str = ""
    name: str = ""

    def validate(self) -> None:
        if self.r == 0:
            raise InvalidArgument("DatasetSpec: rank must be >= 1")
        if DatasetKind(self.kind) == DatasetKind.file:
            if not self.path:
                raise InvalidArgument("DatasetSpec: file dataset needs a path")
            return
        if self.m == 0 or self.n == 0:
            raise InvalidArgument("DatasetSpec: dimensions must be >= 1")
        if self.r > min(self.m, self.n):
            raise InvalidArgument("DatasetSpec: rank exceeds min(m, n)")


def sanitize_label(s: str) -> str:
    """bench.hpp:87-95: anything but [A-Za-z0-9_-] becomes '-' (byte-wise)."""
    out = []
    for b in s.encode():
        c = chr(b)
        ok = ("a" <= c <= "z") or ("A" <= c <= "Z") or ("0" <= c <= "9") or c in "-_"
        out.append(c if ok else "-")
    return "".join(out)


def dataset_label(d: DatasetSpec, index: int) -> str:
    """bench.hpp:97-100."""
    if d.name:
        return sanitize_label(d.name)
    return f"{DatasetKind(d.kind).value}{index}"


@dataclass
class AlgorithmSpec:
    """enmf::AlgorithmSpec (bench.hpp:102-105)."""
    name: str
    config: SolverConfig


def make_algorithm(name: str) -> AlgorithmSpec:
    """bench.hpp:137-139 (presets: algorithm_config, bench.hpp:108-135)."""
    return AlgorithmSpec(name, algorithm_config(name))


def default_algorithms() -> List[str]:
    """bench.hpp:141-145."""
    return ["anls", "e-anls-hp1", "e-anls-hp3", "ahals", "e-ahals-hp1", "e-ahals-hp3"]


@dataclass
class Budget:
    """enmf::Budget (bench.hpp:147-150)."""
    max_iterations: int = 100
    max_seconds: float = math.inf


@dataclass
class SuiteSpec:
    """enmf::SuiteSpec (bench.hpp:152-174).  `threads` = device contexts in flight (0 = 16);
    `precision` and `device` select the device arithmetic and GPU (no reference analogue)."""
    datasets: List[DatasetSpec] = field(default_factory=list)
    algorithms: List[AlgorithmSpec] = field(default_factory=list)
    inits_per_dataset: int = 10
    budget: Budget = field(default_factory=Budget)
    base_seed: int = 1
    threads: int = 1
    wall_timing: bool = False
    precision: Precision = Precision.fp64
    device: int = -1

    def validate(self) -> None:
        if not self.datasets:
            raise InvalidArgument("SuiteSpec: need at least one dataset")
        if not self.algorithms:
            raise InvalidArgument("SuiteSpec: need at least one algorithm")
        if self.inits_per_dataset == 0:
            raise InvalidArgument("SuiteSpec: inits_per_dataset must be >= 1")
        if not (self.budget.max_seconds > 0.0):
            raise InvalidArgument("SuiteSpec: max_seconds must be > 0")
        for d in self.datasets:
            d.validate()


@dataclass
class RunResult:
    """enmf::RunResult (bench.hpp:176-183)."""
    dataset_index: int = 0
    init_index: int = 0
    algorithm_index: int = 0
    record: RunRecord = field(default_factory=RunRecord)
    failed: bool = False
    failure: str = ""


@dataclass
class SuiteResults:
    """enmf::SuiteResults (bench.hpp:185-195); runs in canonical (dataset, init, algorithm) order."""
    spec: SuiteSpec
    runs: List[RunResult] = field(default_factory=list)

    def failed_count(self) -> int:
        return sum(1 for r in self.runs if r.failed)


DataMatrix = Union[np.ndarray, io.SparseMatrix]


def data_rows(x: DataMatrix) -> int:
    return x.rows if isinstance(x, io.SparseMatrix) else int(x.shape[0])


def data_cols(x: DataMatrix) -> int:
    return x.cols if isinstance(x, io.SparseMatrix) else int(x.shape[1])


def load_dataset(d: DatasetSpec) -> DataMatrix:
    """enmf::load_dataset (bench.hpp:207-231)."""
    d.validate()
    kind = DatasetKind(d.kind)
    if kind == DatasetKind.lowrank:
        return io.gen_lowrank(d.m, d.n, d.r, d.seed)
    if kind == DatasetKind.fullrank:
        return io.gen_fullrank(d.m, d.n, d.seed)
    ext = os.path.splitext(d.path)[1]
    if ext in (".mtx", ".mm"):
        x = io.read_matrix_market(d.path)
    elif ext == ".csv":
        x = io.read_dense_csv(d.path)
    else:
        raise UnsupportedFormat(f"cannot infer format of '{d.path}' (expected .mtx, .mm or .csv)")
    if d.r > min(data_rows(x), data_cols(x)):
        raise InvalidArgument(f"DatasetSpec: rank exceeds min dimension of '{d.path}'")
    return x


def _load(ctx: Context, x: DataMatrix) -> None:
    if isinstance(x, io.SparseMatrix):
        ctx.load_csr(x.offsets, x.col_indices, x.values, x.rows, x.cols)
    else:
        ctx.load(x)


def run_suite(spec: SuiteSpec, backend: str = "auto") -> SuiteResults:
    """enmf::run_suite (bench.hpp:233-294) on the GPU.  Load-time errors (a missing or
    malformed file) are raised; per-run failures are captured in RunResult.

    backend "auto": the (dataset, algorithm) groups that fit the packed kernel (dense data, FP64
    presets (HALS or BPP), small shapes, no wall clock — enmf.batch_eligible) run all their inits in ONE
    launch (run_batch_packed); everything else — and every run with backend "streams" — runs
    on per-run device contexts, computed exactly as `run` computes it."""
    spec.validate()
    data = [load_dataset(d) for d in spec.datasets]
    wall = spec.wall_timing or math.isfinite(spec.budget.max_seconds)
    tm = TimingMode.wall if wall else TimingMode.none
    nd, ni, na = len(spec.datasets), spec.inits_per_dataset, len(spec.algorithms)
    total = nd * ni * na
    out = SuiteResults(spec=spec, runs=[RunResult() for _ in range(total)])
    inits = {}

    def init_pair(d, i):
        if (d, i) not in inits:
            inits[(d, i)] = io.random_init(data_rows(data[d]), data_cols(data[d]), spec.datasets[d].r,
                                           io.mix_seed(spec.base_seed, d, i))
        return inits[(d, i)]

    done = set()
    if backend == "auto" and tm == TimingMode.none:
        for d in range(nd):
            if isinstance(data[d], io.SparseMatrix):
                continue
            x = np.asarray(data[d], dtype=np.float64)
            for a in range(na):
                cfg = replace(spec.algorithms[a].config, max_outer_iterations=spec.budget.max_iterations,
                              max_seconds=spec.budget.max_seconds, precision=spec.precision)
                try:
                    cfg.validate()
                except Exception:  # noqa: BLE001 — reported per run by the general path
                    continue
                if not batch_eligible(x.shape[0], x.shape[1], spec.datasets[d].r, cfg):
                    continue
                ts = [(d * ni + i) * na + a for i in range(ni)]
                res = run_batch_packed([(x, *init_pair(d, i)) for i in range(ni)], cfg, spec.device,
                                       raise_errors=False)
                for i, (t, rec) in enumerate(zip(ts, res)):
                    rr = out.runs[t]
                    rr.dataset_index, rr.init_index, rr.algorithm_index = d, i, a
                    if isinstance(rec, Exception):
                        rr.failed, rr.failure = True, str(rec)
                    else:
                        rr.record = rec
                    done.add(t)
    todo = [t for t in range(total) if t not in done]
    if not todo:
        return out
    width = max(1, min(len(todo), spec.threads if spec.threads > 0 else 16))
    pool = [Context(spec.device) for _ in range(width)]
    loaded: List[Optional[int]] = [None] * width
    try:
        for start in range(0, len(todo), width):
            live = []
            for k, t in enumerate(todo[start:start + width]):
                a, i, d = t % na, (t // na) % ni, t // (na * ni)
                rr = out.runs[t]
                rr.dataset_index, rr.init_index, rr.algorithm_index = d, i, a
                try:
                    w0, h0 = init_pair(d, i)
                    cfg = replace(spec.algorithms[a].config, max_outer_iterations=spec.budget.max_iterations,
                                  max_seconds=spec.budget.max_seconds, precision=spec.precision)
                    cfg.validate()
                    ctx = pool[k]
                    if loaded[k] != d:
                        loaded[k] = None
                        _load(ctx, data[d])
                        loaded[k] = d
                    ctx.begin(w0, h0, cfg, tm)
                    ctx.step(int(cfg.max_outer_iterations))
                    live.append((k, t, w0.shape, h0.shape))
                except Exception as e:  # noqa: BLE001 — captured per run (bench.hpp:268-271)
                    rr.failed, rr.failure = True, str(e)
            for k, t, ws, hs in live:
                rr = out.runs[t]
                ctx = pool[k]
                try:
                    recs = ctx.sync()
                    w, h = np.empty(ws), np.empty(hs)
                    nx = ctx.end(w.ctypes.data, h.ctypes.data)
                    rr.record = RunRecord(recs, FactorPair(w, h), nx)
                except Exception as e:  # noqa: BLE001
                    rr.failed, rr.failure = True, str(e)
    finally:
        for ctx in pool:
            ctx.close()
    return out


# ------------------------------------------------------------------ curves
class EminPolicy(enum.Enum):
    zero = 0
    shared_best = 1


@dataclass
class CurvePoint:
    iteration: int = 0
    elapsed_seconds: float = 0.0
    e: float = 0.0


@dataclass
class RunCurve:
    dataset_index: int = 0
    init_index: int = 0
    algorithm_index: int = 0
    points: List[CurvePoint] = field(default_factory=list)


@dataclass
class AlgorithmCurve:
    algorithm_index: int = 0
    points: List[CurvePoint] = field(default_factory=list)


@dataclass
class CurveSet:
    e_min: float = 0.0
    per_run: List[RunCurve] = field(default_factory=list)
    per_algorithm: List[AlgorithmCurve] = field(default_factory=list)


def compute_curves(selected: Sequence[Optional[RunResult]], policy: EminPolicy) -> CurveSet:
    """enmf::compute_curves (bench.hpp:331-399): E(k) = rel_err − e_min per run, and the
    per-algorithm mean with shorter runs padded by their last point."""
    cs = CurveSet()
    ok = [r for r in selected if r is not None and not r.failed and r.record.iterations]
    if policy == EminPolicy.shared_best:
        if any(r.dataset_index != ok[0].dataset_index for r in ok):
            raise MixedDatasets("compute_curves: shared_best floor across different datasets")
        e_min = math.inf
        for r in ok:
            e_min = min(e_min, r.record.final_relative_error())
        cs.e_min = e_min if math.isfinite(e_min) else 0.0
    for r in ok:
        cs.per_run.append(RunCurve(r.dataset_index, r.init_index, r.algorithm_index,
                                   [CurvePoint(it.iteration, it.elapsed_seconds, it.relative_error - cs.e_min)
                                    for it in r.record.iterations]))
    for a in sorted({rc.algorithm_index for rc in cs.per_run}):
        group = [rc for rc in cs.per_run if rc.algorithm_index == a]
        length = max(len(rc.points) for rc in group)
        ac = AlgorithmCurve(a, [])
        for p in range(length):
            esum = tsum = 0.0
            for rc in group:
                cp = rc.points[p] if p < len(rc.points) else rc.points[-1]
                esum += cp.e
                tsum += cp.elapsed_seconds
            ac.points.append(CurvePoint(p, tsum / len(group), esum / len(group)))
        cs.per_algorithm.append(ac)
    return cs


def compute_curves_for_dataset(res: SuiteResults, dataset_index: int) -> CurveSet:
    """bench.hpp:401-415: zero floor for exact low-rank synthetics, shared best otherwise."""
    sel = [r for r in res.runs if r.dataset_index == dataset_index]
    kind = DatasetKind(res.spec.datasets[dataset_index].kind)
    return compute_curves(sel, EminPolicy.zero if kind == DatasetKind.lowrank else EminPolicy.shared_best)


# ------------------------------------------------------------------ ranking
@dataclass
class RankingRow:
    algorithm: str = ""
    mean_final_rel_err: float = 0.0
    std_final_rel_err: float = 0.0
    ranking: List[int] = field(default_factory=list)


@dataclass
class RankingTable:
    rows: List[RankingRow] = field(default_factory=list)
    group_count: int = 0
    tie_groups: int = 0


def rank_final_errors(res: SuiteResults) -> RankingTable:
    """enmf::rank_final_errors (bench.hpp:438-480): per (dataset, init) group a stable
    sort of the final errors awards placements; sample mean / std per algorithm."""
    spec = res.spec
    na, ni, nd = len(spec.algorithms), spec.inits_per_dataset, len(spec.datasets)
    table = RankingTable(rows=[RankingRow(a.name, 0.0, 0.0, [0] * na) for a in spec.algorithms])
    finals: List[List[float]] = [[] for _ in range(na)]
    for d in range(nd):
        for i in range(ni):
            errs = []
            for a in range(na):
                rr = res.runs[(d * ni + i) * na + a]
                if rr.failed or not rr.record.iterations:
                    raise MissingRun(f"rank_final_errors: no result for dataset {d}, init {i}, algorithm "
                                     f"'{spec.algorithms[a].name}'" + (f": {rr.failure}" if rr.failed else ""))
                errs.append(rr.record.final_relative_error())
                finals[a].append(errs[a])
            order = sorted(range(na), key=lambda k: errs[k])   # stable, like std::stable_sort
            tied = False
            for pos, a in enumerate(order):
                table.rows[a].ranking[pos] += 1
                if pos > 0 and errs[a] == errs[order[pos - 1]]:
                    tied = True
            table.tie_groups += 1 if tied else 0
            table.group_count += 1
    for a in range(na):
        v = finals[a]
        mean = 0.0
        for x in v:
            mean += x
        mean /= len(v)
        var = 0.0
        for x in v:
            var += (x - mean) * (x - mean)
        table.rows[a].mean_final_rel_err = mean
        table.rows[a].std_final_rel_err = math.sqrt(var / (len(v) - 1)) if len(v) > 1 else 0.0
    return table


# ------------------------------------------------------------------ artifacts
@dataclass
class EmitOptions:
    run_csv: bool = True
    curve_csv: bool = True
    summary_json: bool = True


def dataset_error_floors(res: SuiteResults) -> List[float]:
    """bench.hpp:493-507: 0 for low-rank synthetics, else the best final error of the pool."""
    floors = [0.0] * len(res.spec.datasets)
    for d, ds in enumerate(res.spec.datasets):
        if DatasetKind(ds.kind) == DatasetKind.lowrank:
            continue
        best = math.inf
        for r in res.runs:
            if r.dataset_index == d and not r.failed and r.record.iterations:
                best = min(best, r.record.final_relative_error())
        floors[d] = best if math.isfinite(best) else 0.0
    return floors


def _json_number(v: float) -> str:
    """A double as nlohmann::json::dump writes it: the shortest round-trip digits, fixed
    notation while the decimal point position n lies in (-4, 15], else d.ddde±XX (two
    exponent digits at least); integral values get '.0'; non-finite values are null."""
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    r = repr(abs(v))
    m, _, e = r.partition("e")
    ip, _, fp = m.partition(".")
    digits, exp10 = ip + fp, (int(e) if e else 0) - len(fp)      # value = int(digits)·10^exp10
    while len(digits) > 1 and digits.endswith("0"):
        digits, exp10 = digits[:-1], exp10 + 1
    digits = digits.lstrip("0")
    k, n = len(digits), len(digits) + exp10
    if k <= n <= 15:
        s = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + digits
    else:
        x = n - 1
        s = digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if x < 0 else "+") + f"{abs(x):02d}"
    return ("-" if v < 0 else "") + s


def _dump(obj, indent: int = 0) -> str:
    """nlohmann::ordered_json::dump(2) layout."""
    pad, inner = " " * indent, " " * (indent + 2)
    if obj is None:
        return "null"
    if obj is True:
        return "true"
    if obj is False:
        return "false"
    if isinstance(obj, int):
        return str(obj)
    if isinstance(obj, float):
        return _json_number(obj)
    if isinstance(obj, str):
        return json.dumps(obj, ensure_ascii=False)
    if isinstance(obj, list):
        if not obj:
            return "[]"
        return "[\n" + ",\n".join(inner + _dump(v, indent + 2) for v in obj) + "\n" + pad + "]"
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        return ("{\n" + ",\n".join(inner + json.dumps(k, ensure_ascii=False) + ": " + _dump(v, indent + 2)
                                   for k, v in obj.items()) + "\n" + pad + "}")
    raise TypeError(type(obj))


def emit(res: SuiteResults, out_dir, opts: EmitOptions = EmitOptions()) -> List[str]:
    """enmf::emit (bench.hpp:509-646): run traces, per-algorithm mean curves and a
    summary JSON under out_dir; returns the paths in the order written."""
    try:
        os.makedirs(out_dir, exist_ok=True)
    except OSError as e:
        raise io.IoError(f"cannot create output directory '{out_dir}': {e.strerror}") from e
    spec = res.spec
    written: List[str] = []
    floors = dataset_error_floors(res)
    if opts.run_csv:
        for r in res.runs:
            if r.failed:
                continue
            p = os.path.join(out_dir, f"run_{dataset_label(spec.datasets[r.dataset_index], r.dataset_index)}_"
                                      f"{sanitize_label(spec.algorithms[r.algorithm_index].name)}_{r.init_index}.csv")
            io.write_run_csv(p, r.record, floors[r.dataset_index])
            written.append(p)
    if opts.curve_csv:
        for d in range(len(spec.datasets)):
            cs = compute_curves_for_dataset(res, d)
            for ac in cs.per_algorithm:
                p = os.path.join(out_dir, f"curve_{dataset_label(spec.datasets[d], d)}_"
                                          f"{sanitize_label(spec.algorithms[ac.algorithm_index].name)}.csv")
                lines = ["iter,elapsed_s,E_mean\n"]
                for cp in ac.points:
                    lines.append(f"{cp.iteration},{io.format_double(cp.elapsed_seconds)},{io.format_double(cp.e)}\n")
                try:
                    with open(p, "w", newline="") as f:
                        f.write("".join(lines))
                except OSError as e:
                    raise io.IoError(f"cannot open '{p}' for writing") from e
                written.append(p)
    if opts.summary_json:
        j = {"base_seed": int(spec.base_seed), "inits_per_dataset": int(spec.inits_per_dataset),
             "budget": {"max_iterations": int(spec.budget.max_iterations),
                        "max_seconds": float(spec.budget.max_seconds)
                        if math.isfinite(spec.budget.max_seconds) else None}}
        dsl = []
        for d, ds in enumerate(spec.datasets):
            jd = {"label": dataset_label(ds, d), "kind": DatasetKind(ds.kind).value}
            if DatasetKind(ds.kind) == DatasetKind.file:
                jd["path"] = ds.path
            else:
                jd["m"], jd["n"], jd["seed"] = int(ds.m), int(ds.n), int(ds.seed)
            jd["rank"] = int(ds.r)
            jd["e_min"] = float(floors[d])
            dsl.append(jd)
        j["datasets"] = dsl
        al = []
        for a in spec.algorithms:
            c = a.config
            ja = {"name": a.name, "inner_h": "exact" if int(c.inner_h) == 0 else "hals",
                  "inner_w": "exact" if int(c.inner_w) == 0 else "hals",
                  "extrapolation": bool(c.extrapolation_enabled)}
            if c.extrapolation_enabled:
                ja.update(hp=int(c.hp), beta0=float(c.beta0), gamma=float(c.gamma), gamma_bar=float(c.gamma_bar),
                          eta=float(c.eta))
            al.append(ja)
        j["algorithms"] = al
        rl = []
        for r in res.runs:
            jr = {"dataset": dataset_label(spec.datasets[r.dataset_index], r.dataset_index), "init": r.init_index,
                  "algorithm": spec.algorithms[r.algorithm_index].name}
            if r.failed:
                jr["failed"], jr["error"] = True, r.failure
            else:
                its = r.record.iterations
                jr["failed"] = False
                jr["iterations"] = int(its[-1].iteration) if its else 0
                jr["final_rel_err"] = float(r.record.final_relative_error())
                jr["restarts"] = sum(1 for it in its if it.restarted)
            rl.append(jr)
        j["runs"] = rl
        if res.failed_count() == 0:
            table = rank_final_errors(res)
            j["ranking"] = [{"algorithm": row.algorithm, "mean_final_rel_err": float(row.mean_final_rel_err),
                             "std_final_rel_err": float(row.std_final_rel_err), "ranking": list(row.ranking)}
                            for row in table.rows]
            j["group_count"] = table.group_count
            j["tie_groups"] = table.tie_groups
        else:
            j["ranking"] = None
            j["failed_runs"] = res.failed_count()
        p = os.path.join(out_dir, "summary.json")
        try:
            with open(p, "w", newline="") as f:
                f.write(_dump(j) + "\n")
        except OSError as e:
            raise io.IoError(f"cannot open '{p}' for writing") from e
        written.append(p)
    return written

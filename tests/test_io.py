"""CPU tier: the data formats and generators of csrc/io.cpp against the reference.

Pinned two ways: (1) the committed fixtures tests/golden/io.json, produced by the
reference's own data.hpp (tests/golden/make_golden_io.py via oracle/_ref); (2) where
oracle/_ref/libenmf_ref_io.so exists, live differential fuzzing of both readers on
mutated files.  Bar: bit-identical arrays, identical error class, message and line.
Modelled on the reference's test_data.cpp and acceptance.cpp round trips.
"""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

import io_corpus as K
from paper_1805_06604_b200 import data as D
from paper_1805_06604_b200 import enmf as E

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "io.json")))
CODE = {E.ParseError: 7, E.UnsupportedFormat: 8, E.IoError: 9, E.InvalidArgument: 1}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_IO = os.path.join(ROOT, "oracle", "_ref", "libenmf_ref_io.so")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(fn, path, full=True):
    try:
        x = fn(path)
    except (E.ParseError, E.UnsupportedFormat, E.IoError, E.InvalidArgument) as e:
        return {"code": CODE[type(e)], "msg": str(e), "line": getattr(e, "line", 0)}
    if isinstance(x, D.SparseMatrix):
        out = {"rows": x.rows, "cols": x.cols, "nnz": x.nnz}
        if full:
            out.update(offsets=x.offsets.tolist(), col_idx=x.col_indices.tolist(),
                       values=[float(v).hex() for v in x.values])
        else:
            out.update(sha_offsets=sha(x.offsets.astype(np.uint64)), sha_idx=sha(x.col_indices.astype(np.uint64)),
                       sha_values=sha(x.values))
        return out
    out = {"rows": x.shape[0], "cols": x.shape[1]}
    if full:
        out["values"] = [float(v).hex() for v in x.ravel()]
    else:
        out["sha_values"] = sha(x.ravel())
    return out


@pytest.mark.parametrize("name", sorted(K.MM_CASES))
def test_matrix_market_case_matches_reference(tmp_path, name):
    p = tmp_path / (name + ".mtx")
    p.write_bytes(K.MM_CASES[name].encode())
    assert outcome(D.read_matrix_market, p) == GOLDEN["mm"][name]


def test_matrix_market_missing_file_is_io_error(tmp_path):
    got = outcome(D.read_matrix_market, tmp_path / "does-not-exist.mtx")
    got["msg"] = got["msg"].replace(str(tmp_path), "<dir>")
    assert got == GOLDEN["mm"]["missing_file"]


@pytest.mark.parametrize("name", sorted(K.CSV_CASES))
def test_dense_csv_case_matches_reference(tmp_path, name):
    p = tmp_path / (name + ".csv")
    p.write_bytes(K.CSV_CASES[name].encode())
    assert outcome(D.read_dense_csv, p) == GOLDEN["csv"][name]


@pytest.mark.parametrize("name,seed,kind", K.BIG_MM)
def test_large_matrix_market_parallel_path(tmp_path, name, seed, kind):
    """Files above the 1 MiB threshold parse on all host threads; errors deep inside
    still report the reference's first error and line."""
    p = tmp_path / (name + ".mtx")
    p.write_bytes(K.big_mm(seed, kind).encode())
    assert os.path.getsize(p) > (1 << 20)
    assert outcome(D.read_matrix_market, p, full=False) == GOLDEN["big_mm"][name]


@pytest.mark.parametrize("name,seed,kind", K.BIG_CSV)
def test_large_dense_csv_parallel_path(tmp_path, name, seed, kind):
    p = tmp_path / (name + ".csv")
    p.write_bytes(K.big_csv(seed, kind).encode())
    assert os.path.getsize(p) > (1 << 20)
    assert outcome(D.read_dense_csv, p, full=False) == GOLDEN["big_csv"][name]


def test_format_double_matches_reference():
    for hx, s in GOLDEN["format"]:
        assert D.format_double(float.fromhex(hx)) == s
        assert float(s) == float.fromhex(hx)          # round trip (test_data.cpp:95-115)


def test_run_csv_matches_reference(tmp_path):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden_io import records
    for name, (rows, e_min) in records().items():
        rec = E.RunRecord([E.IterationRecord(it, el, e, rel, beta, bool(rs)) for it, el, e, rel, beta, rs in rows])
        p = tmp_path / (name + ".csv")
        D.write_run_csv(p, rec, e_min)
        assert p.read_bytes().decode() == GOLDEN["run_csv"][name]
    # the reference test's exact lines (test_data.cpp:289-296)
    lines = GOLDEN["run_csv"]["ref_test"].splitlines()
    assert lines == ["iter,elapsed_s,rel_err,E,beta,restarted", "0,0,0.5,0.45,0.5,0",
                     "1,0.25,0.2,0.15000000000000002,0.55,1"]


def test_writers_match_reference(tmp_path):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden_io import write_matrices
    for name, d in write_matrices().items():
        p = tmp_path / (name + ".mtx")
        D.write_matrix_market(p, D.SparseMatrix.from_dense(d))
        t = p.read_bytes().decode()
        assert (t if name == "small" else hashlib.sha256(t.encode()).hexdigest()) == GOLDEN["write_mm"][name]
        p = tmp_path / (name + ".csv")
        D.write_dense_csv(p, d)
        t = p.read_bytes().decode()
        assert (t if name == "small" else hashlib.sha256(t.encode()).hexdigest()) == GOLDEN["write_csv"][name]


def test_generators_match_reference():
    for key, want in GOLDEN["gen"].items():
        m, n, r, seed = map(int, key.split("_"))
        assert sha(D.gen_lowrank(m, n, r, seed)) == want["gen_lowrank"]
        assert [sha(a) for a in D.random_init(m, n, r, seed + 1)] == want["random_init"]
        assert [sha(a) for a in D.lowrank_factors(m, n, r, seed + 2)] == want["lowrank_factors"]
        assert sha(D.gen_fullrank(m, n, seed + 3)) == want["gen_fullrank"]
    for b, a, c, h in GOLDEN["mix_seed"]:
        assert D.mix_seed(b, a, c) == h
    with pytest.raises(E.InvalidArgument):
        D.lowrank_factors(4, 3, 4, 1)
    with pytest.raises(E.InvalidArgument):
        D.gen_lowrank(4, 3, 0, 1)


def test_roundtrips_are_lossless(tmp_path):
    """test_data.cpp:117-131, 229-236 and acceptance.cpp dense/sparse/large round trips."""
    rng = np.random.default_rng(149)
    for rep in range(8):
        m, n = int(rng.integers(1, 40)), int(rng.integers(1, 25))
        x = np.ldexp(rng.uniform(-1, 1, (m, n)), rng.integers(-20, 20, (m, n)))
        D.write_dense_csv(tmp_path / "d.csv", x)
        assert np.array_equal(D.read_dense_csv(tmp_path / "d.csv"), x)
        x[rng.random(x.shape) < 0.7] = 0.0
        s = D.SparseMatrix.from_dense(x)
        D.write_matrix_market(tmp_path / "s.mtx", s)
        y = D.read_matrix_market(tmp_path / "s.mtx")
        assert np.array_equal(y.offsets, s.offsets) and np.array_equal(y.col_indices, s.col_indices)
        assert np.array_equal(y.values, s.values) and np.array_equal(y.to_dense(), x)
    # corpus scale: k -> (k mod m, k mod n) distinct because m, n are coprime (acceptance.cpp:452-470)
    m, n, count = 7094, 41681, 223839
    k = np.arange(count, dtype=np.uint64)
    vals = rng.uniform(0.1, 5.0, count)
    s = D.SparseMatrix.from_triplets(m, n, list(zip((k % m).tolist(), (k % n).tolist(), vals.tolist())))
    D.write_matrix_market(tmp_path / "big.mtx", s)
    y = D.read_matrix_market(tmp_path / "big.mtx")
    assert y.nnz == count and np.array_equal(y.offsets, s.offsets)
    assert np.array_equal(y.col_indices, s.col_indices) and np.array_equal(y.values, s.values)


def test_writer_rejects_invalid_csr(tmp_path):
    bad = D.SparseMatrix(2, 2, np.array([0, 2, 2], np.uint64), np.array([1, 0], np.uint64), np.array([1.0, 2.0]))
    with pytest.raises(E.InvalidArgument, match="strictly increasing"):
        D.write_matrix_market(tmp_path / "x.mtx", bad)
    with pytest.raises(E.IoError):
        D.write_dense_csv(tmp_path / "no" / "such" / "dir.csv", np.ones((2, 2)))


# ------------------------------------------------------- live differential fuzzing
def _ref_lib():
    if not os.path.exists(REF_IO):
        pytest.skip("oracle/_ref/libenmf_ref_io.so not built here")
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import make_golden_io as G
    return G, G.lib()


def _mutate(rng, text):
    b = bytearray(text.encode())
    for _ in range(int(rng.integers(1, 4))):
        op = int(rng.integers(0, 4))
        pos = int(rng.integers(0, max(1, len(b))))
        if op == 0 and b:
            del b[pos]
        elif op == 1:
            b.insert(pos, rng.choice(list(b" \n\t,.-+e%x0123456789\r")))
        elif op == 2 and b:
            b[pos] = rng.choice(list(b" \n,.-e0123456789"))
        else:
            b[pos:pos] = b"\n"
    return bytes(b)


def test_fuzz_readers_against_reference(tmp_path):
    G, L = _ref_lib()
    rng = np.random.default_rng(2026)
    seeds = list(K.MM_CASES.values())
    for t in range(400):
        data = _mutate(rng, seeds[t % len(seeds)])
        p = tmp_path / "f.mtx"
        p.write_bytes(data)
        assert outcome(D.read_matrix_market, p) == G.read_mm(L, str(p), True), data
    seeds = list(K.CSV_CASES.values())
    for t in range(300):
        data = _mutate(rng, seeds[t % len(seeds)])
        p = tmp_path / "f.csv"
        p.write_bytes(data)
        assert outcome(D.read_dense_csv, p) == G.read_csv(L, str(p), True), data


def test_fuzz_large_files_against_reference(tmp_path):
    """Mutations inside large files: the parallel path must fall back to the exact error."""
    G, L = _ref_lib()
    rng = np.random.default_rng(77)
    base = K.big_mm(31, "ok").encode()
    for t in range(6):
        b = bytearray(base)
        pos = int(rng.integers(len(b) // 2, len(b)))
        b[pos:pos + 1] = [b"x", b"\n", b" 7", b"", b"\n\n5 5 1\n"][t % 5]
        p = tmp_path / "g.mtx"
        p.write_bytes(bytes(b))
        assert outcome(D.read_matrix_market, p, False) == G.read_mm(L, str(p), False)
    base = K.big_csv(32, "ok").encode()
    for t in range(4):
        b = bytearray(base)
        pos = int(rng.integers(len(b) // 2, len(b)))
        b[pos:pos + 1] = [b",", b"\n", b"e", b""][t]
        p = tmp_path / "g.csv"
        p.write_bytes(bytes(b))
        assert outcome(D.read_dense_csv, p, False) == G.read_csv(L, str(p), False)

"""Golden fixtures for the data formats and the suite harness, from the REFERENCE itself.

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden_io.py
It calls the unmodified reference (enmf/data.hpp, enmf/bench.hpp) compiled in place into
oracle/_ref/libenmf_ref_io.so by oracle/ref_io_shim.cpp, on the inputs of tests/io_corpus.py,
and writes tests/golden/io.json plus tests/golden/suite/ (the reference's emit() output for
the suite spec in tests/golden/suite/spec.json).  The GPU box only reads these files.
"""
import ctypes as C
import hashlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import io_corpus as K  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
IO_SO = os.path.join(ROOT, "oracle", "_ref", "libenmf_ref_io.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libenmf_ref.so")


class CIter(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("elapsed_seconds", C.c_double), ("error", C.c_double),
                ("relative_error", C.c_double), ("beta", C.c_double), ("restarted", C.c_int32),
                ("inner_h_count", C.c_int32), ("inner_w_count", C.c_int32), ("reinit_events", C.c_int32)]


def lib():
    L = C.CDLL(IO_SO)
    sz, u64pp, dpp = C.c_size_t, C.POINTER(C.POINTER(C.c_uint64)), C.POINTER(C.POINTER(C.c_double))
    L.ref_io_last_error.restype = C.c_char_p
    L.ref_io_last_line.restype = sz
    L.ref_io_free.argtypes = [C.c_void_p]
    L.ref_io_read_mm.argtypes = [C.c_char_p, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz), u64pp, u64pp, dpp]
    L.ref_io_read_csv.argtypes = [C.c_char_p, C.POINTER(sz), C.POINTER(sz), dpp]
    L.ref_io_write_mm.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p, sz, sz]
    L.ref_io_write_csv.argtypes = [C.c_char_p, C.c_void_p, sz, sz]
    L.ref_io_write_run_csv.argtypes = [C.c_char_p, C.POINTER(CIter), sz, C.c_double]
    L.ref_io_format_double.argtypes = [C.c_double, C.c_char_p, sz]
    L.ref_io_format_double.restype = sz
    L.ref_gen_fullrank.argtypes = [sz, sz, C.c_uint64, C.c_void_p]
    L.ref_lowrank_factors.argtypes = [sz, sz, sz, C.c_uint64, C.c_void_p, C.c_void_p]
    L.ref_suite_emit.argtypes = [C.c_char_p, C.c_char_p]
    return L


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def err(L, rc):
    return {"code": rc, "msg": L.ref_io_last_error().decode(), "line": int(L.ref_io_last_line())}


def read_mm(L, path, full):
    rows, cols, nnz = C.c_size_t(), C.c_size_t(), C.c_size_t()
    off, idx, val = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)(), C.POINTER(C.c_double)()
    rc = L.ref_io_read_mm(path.encode(), C.byref(rows), C.byref(cols), C.byref(nnz), C.byref(off), C.byref(idx),
                          C.byref(val))
    if rc:
        return err(L, rc)
    m, k = rows.value, nnz.value
    o = np.ctypeslib.as_array(off, (m + 1,)).copy()
    i = np.ctypeslib.as_array(idx, (max(k, 1),))[:k].copy()
    v = np.ctypeslib.as_array(val, (max(k, 1),))[:k].copy()
    for p in (off, idx, val):
        L.ref_io_free(C.cast(p, C.c_void_p))
    out = {"rows": m, "cols": cols.value, "nnz": k}
    if full:
        out.update(offsets=o.tolist(), col_idx=i.tolist(), values=[float(x).hex() for x in v])
    else:
        out.update(sha_offsets=sha(o.astype(np.uint64)), sha_idx=sha(i.astype(np.uint64)), sha_values=sha(v))
    return out


def read_csv(L, path, full):
    rows, cols = C.c_size_t(), C.c_size_t()
    val = C.POINTER(C.c_double)()
    rc = L.ref_io_read_csv(path.encode(), C.byref(rows), C.byref(cols), C.byref(val))
    if rc:
        return err(L, rc)
    v = np.ctypeslib.as_array(val, (rows.value * cols.value,)).copy()
    L.ref_io_free(C.cast(val, C.c_void_p))
    out = {"rows": rows.value, "cols": cols.value}
    if full:
        out["values"] = [float(x).hex() for x in v]
    else:
        out["sha_values"] = sha(v)
    return out


def text_of(path):
    with open(path, "rb") as f:
        return f.read().decode()


def records():
    """The reference test's trace (test_data.cpp:269-303) and a longer synthetic one."""
    a = [(0, 0.0, 5.0, 0.5, 0.5, 0), (1, 0.25, 2.0, 0.2, 0.55, 1)]
    rng = np.random.default_rng(5)
    b = [(k, float(rng.uniform(0, 3)) * k, float(rng.uniform(0, 9)), float(rng.uniform(0, 1)),
          float(rng.uniform(0, 1)), int(rng.integers(0, 2))) for k in range(40)]
    return {"ref_test": (a, 0.05), "synthetic": (b, 0.0123)}


def to_citers(rows):
    arr = (CIter * max(1, len(rows)))()
    for k, (it, el, e, rel, beta, rs) in enumerate(rows):
        arr[k].iteration, arr[k].elapsed_seconds, arr[k].error = it, el, e
        arr[k].relative_error, arr[k].beta, arr[k].restarted = rel, beta, rs
    return arr


def write_matrices():
    rng = np.random.default_rng(77)
    d = rng.standard_normal((9, 7)) * np.exp(rng.uniform(-10, 10, (9, 7)))
    d[rng.random(d.shape) < 0.6] = 0.0
    big = rng.standard_normal((3000, 200))
    big[rng.random(big.shape) < 0.5] = 0.0
    return {"small": d, "big": big}


def csr_of(d):
    i, j = np.nonzero(d)
    off = np.zeros(d.shape[0] + 1, dtype=np.uint64)
    np.add.at(off, i + 1, 1)
    return np.cumsum(off, dtype=np.uint64), j.astype(np.uint64), d[i, j].copy()


SUITE_SPEC = {
    "datasets": [
        {"kind": "lowrank", "m": 40, "n": 32, "r": 4, "seed": 500},
        {"kind": "fullrank", "m": 30, "n": 24, "r": 3, "seed": 501, "name": "uniform noise"},
        {"kind": "file", "r": 3, "path": "docs.mtx"},
        {"kind": "file", "r": 2, "path": "faces.csv", "name": "faces"},
    ],
    "algorithms": ["anls", "e-anls-hp1", "e-anls-hp3", "ahals", "e-ahals-hp1", "e-ahals-hp3"],
    "inits_per_dataset": 2, "max_iterations": 30, "base_seed": 13, "threads": 4, "wall_timing": False,
}


def suite_inputs(dirpath):
    """docs.mtx: a small tf-idf-like term × document matrix; faces.csv: a dense nonnegative
    image-like matrix (both seeded synthetics written by the reference's own writers)."""
    L = lib()
    rng = np.random.default_rng(9)
    m, n = 60, 25
    d = np.zeros((m, n))
    for j in range(n):
        terms = rng.choice(m, size=int(rng.integers(4, 15)), replace=False)
        d[terms, j] = rng.integers(1, 5, terms.size) * np.log(n / rng.integers(1, n, terms.size) + 1.0)
        d[:, j] /= np.linalg.norm(d[:, j])
    off, idx, val = csr_of(d)
    assert L.ref_io_write_mm(os.path.join(dirpath, "docs.mtx").encode(), off.ctypes.data, idx.ctypes.data,
                             val.ctypes.data, m, n) == 0
    f = rng.uniform(0, 1, (20, 16)) @ rng.uniform(0, 1, (16, 18)) / 16.0
    assert L.ref_io_write_csv(os.path.join(dirpath, "faces.csv").encode(), f.ctypes.data, 20, 18) == 0


def stock_nlohmann_layout(text: str) -> str:
    """The json.hpp available here is cudnn-frontend's copy of nlohmann 3.11.3, patched to
    print integer arrays on one line ("Custom from FE", json.hpp:20609-20613); the reference
    vendors the stock 3.11.3 (README.md:50), which prints every array one element per line.
    Restore the stock layout so the fixture is what the reference's own build emits."""
    import re

    def expand(m):
        pad, key, items = m.group(1), m.group(2), m.group(3).split(",")
        inner = pad + "  "
        return f"{pad}{key}[\n" + ",\n".join(inner + v for v in items) + f"\n{pad}]"
    return re.sub(r"^( *)(\"[^\"]*\": )\[(-?\d+(?:,-?\d+)*)\]", expand, text, flags=re.M)


def linesearch_cases():
    """Inputs for optimal_beta_linesearch (engine.hpp:522-540), after test_engine.cpp:493-539:
    random small cases, a zero-residual case, a larger one, a CSR X and a zero direction."""
    rng = np.random.default_rng(127)
    cases = []
    for k in range(10):
        m, n, r = 10, 9, 3
        cases.append(("small%d" % k, rng.random((m, n)), rng.random((m, r)), rng.random((m, r)), rng.random((r, n))))
    wn, w, h = rng.random((9, 3)), rng.random((9, 3)), rng.random((3, 8))
    cases.append(("zero_residual", wn @ h, wn, w, h))
    cases.append(("large", rng.random((300, 257)), rng.random((300, 17)), rng.random((300, 17)),
                  rng.random((17, 257))))
    xs = rng.random((200, 150))
    xs[rng.random(xs.shape) > 0.05] = 0.0
    cases.append(("csr", xs, rng.random((200, 6)), rng.random((200, 6)), rng.random((6, 150))))
    wn = rng.random((8, 2))
    cases.append(("zero_direction", rng.random((8, 7)), wn, wn.copy(), rng.random((2, 7))))
    return cases


def linesearch_golden():
    R = C.CDLL(REF_SO)
    sz, dp = C.c_size_t, C.c_void_p
    R.ref_optimal_beta_linesearch.argtypes = [dp, sz, sz, dp, dp, dp, sz, C.POINTER(C.c_double)]
    R.ref_optimal_beta_linesearch_csr.argtypes = [dp, dp, dp, sz, sz, dp, dp, dp, sz, C.POINTER(C.c_double)]
    out = {}
    for name, x, wn, w, h in linesearch_cases():
        b = C.c_double(0)
        m, n, r = x.shape[0], x.shape[1], wn.shape[1]
        args = [wn.ctypes.data, w.ctypes.data, h.ctypes.data, r, C.byref(b)]
        if name == "csr":
            off, idx, val = csr_of(x)
            rc = R.ref_optimal_beta_linesearch_csr(off.ctypes.data, idx.ctypes.data, val.ctypes.data, m, n, *args)
        else:
            rc = R.ref_optimal_beta_linesearch(x.ctypes.data, m, n, *args)
        out[name] = (rc, b.value)
    np.savez_compressed(os.path.join(OUT, "linesearch.npz"), names=np.array(list(out)),
                        rc=np.array([v[0] for v in out.values()]), beta=np.array([v[1] for v in out.values()]))


def main():
    L = lib()
    R = C.CDLL(REF_SO)
    sz = C.c_size_t
    R.ref_gen_lowrank.argtypes = [sz, sz, sz, C.c_uint64, C.c_void_p]
    R.ref_random_init.argtypes = [sz, sz, sz, C.c_uint64, C.c_void_p, C.c_void_p]
    R.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
    R.ref_mix_seed.restype = C.c_uint64
    g = {"mm": {}, "csv": {}, "big_mm": {}, "big_csv": {}, "format": [], "run_csv": {}, "write_mm": {},
         "write_csv": {}, "gen": {}}
    tmp = tempfile.mkdtemp()
    try:
        for name, text in K.MM_CASES.items():
            p = os.path.join(tmp, name + ".mtx")
            open(p, "wb").write(text.encode())
            g["mm"][name] = read_mm(L, p, True)
        g["mm"]["missing_file"] = read_mm(L, os.path.join(tmp, "does-not-exist.mtx"), True)
        g["mm"]["missing_file"]["msg"] = g["mm"]["missing_file"]["msg"].replace(tmp, "<dir>")
        for name, text in K.CSV_CASES.items():
            p = os.path.join(tmp, name + ".csv")
            open(p, "wb").write(text.encode())
            g["csv"][name] = read_csv(L, p, True)
        for name, seed, kind in K.BIG_MM:
            p = os.path.join(tmp, name + ".mtx")
            open(p, "wb").write(K.big_mm(seed, kind).encode())
            g["big_mm"][name] = read_mm(L, p, False)
        for name, seed, kind in K.BIG_CSV:
            p = os.path.join(tmp, name + ".csv")
            open(p, "wb").write(K.big_csv(seed, kind).encode())
            g["big_csv"][name] = read_csv(L, p, False)
        buf = C.create_string_buffer(64)
        for v in K.format_values():
            n = L.ref_io_format_double(v, buf, 64)
            g["format"].append([float(v).hex(), buf.value[:n].decode()])
        for name, (rows, e_min) in records().items():
            p = os.path.join(tmp, name + ".csv")
            assert L.ref_io_write_run_csv(p.encode(), to_citers(rows), len(rows), e_min) == 0
            g["run_csv"][name] = text_of(p)
        for name, d in write_matrices().items():
            off, idx, val = csr_of(d)
            p = os.path.join(tmp, name + ".mtx")
            assert L.ref_io_write_mm(p.encode(), off.ctypes.data, idx.ctypes.data, val.ctypes.data, *d.shape) == 0
            t = text_of(p)
            g["write_mm"][name] = t if name == "small" else hashlib.sha256(t.encode()).hexdigest()
            dd = np.ascontiguousarray(d)
            p = os.path.join(tmp, name + ".csv")
            assert L.ref_io_write_csv(p.encode(), dd.ctypes.data, *d.shape) == 0
            t = text_of(p)
            g["write_csv"][name] = t if name == "small" else hashlib.sha256(t.encode()).hexdigest()
        for (m, n, r, seed) in [(37, 23, 5, 11), (200, 200, 20, 1), (64, 300, 7, 99)]:
            x = np.empty((m, n))
            R.ref_gen_lowrank(m, n, r, seed, x.ctypes.data)
            w, h = np.empty((m, r)), np.empty((r, n))
            R.ref_random_init(m, n, r, seed + 1, w.ctypes.data, h.ctypes.data)
            wl, hl = np.empty((m, r)), np.empty((r, n))
            assert L.ref_lowrank_factors(m, n, r, seed + 2, wl.ctypes.data, hl.ctypes.data) == 0
            f = np.empty((m, n))
            assert L.ref_gen_fullrank(m, n, seed + 3, f.ctypes.data) == 0
            g["gen"][f"{m}_{n}_{r}_{seed}"] = {"gen_lowrank": sha(x), "random_init": [sha(w), sha(h)],
                                               "lowrank_factors": [sha(wl), sha(hl)], "gen_fullrank": sha(f)}
        g["mix_seed"] = [[b, a, c, int(R.ref_mix_seed(b, a, c))] for b, a, c in
                         [(0, 0, 0), (1, 2, 3), (13, 0, 1), (2 ** 64 - 1, 7, 2 ** 63)]]
    finally:
        shutil.rmtree(tmp)
    with open(os.path.join(OUT, "io.json"), "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)

    linesearch_golden()

    sdir = os.path.join(OUT, "suite")
    shutil.rmtree(sdir, ignore_errors=True)
    os.makedirs(sdir)
    suite_inputs(sdir)
    with open(os.path.join(sdir, "spec.json"), "w") as f:
        json.dump(SUITE_SPEC, f, indent=1)
    cwd = os.getcwd()
    os.chdir(sdir)                     # the file datasets are named relative to the suite dir
    try:
        rc = L.ref_suite_emit(json.dumps(SUITE_SPEC).encode(), b"emit")
        assert rc == 0, L.ref_io_last_error()
        with open(os.path.join("emit", "summary.json")) as f:
            text = stock_nlohmann_layout(f.read())
        with open(os.path.join("emit", "summary.json"), "w") as f:
            f.write(text)
    finally:
        os.chdir(cwd)
    print("wrote", os.path.join(OUT, "io.json"), "and", sdir, len(os.listdir(os.path.join(sdir, "emit"))), "files")


if __name__ == "__main__":
    main()

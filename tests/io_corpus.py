"""Inputs for the data-format parity tests (tests/test_io.py) and their golden fixtures
(tests/golden/make_golden_io.py, which runs the reference's own readers on them).

Small cases are literal file texts: the reference's own test layouts
(test_data.cpp:135-265) and every error branch of read_matrix_market /
read_dense_csv (data.hpp:159-295).  Large cases are generated from a seed so the
multi-threaded path of csrc/io.cpp is exercised (files above its 1 MiB threshold),
with and without an error deep inside the file.
"""
import numpy as np

BANNER = "%%MatrixMarket matrix coordinate real general\n"

MM_CASES = {
    "standard": BANNER + "% a comment between banner and size\n\n3 4 3\n1 1 2.5\n3 2 -1.25e-1\n2 4 7\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 1 3\n2 2 -4\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n",
    "array": "%%MatrixMarket matrix array real general\n2 2\n1.0\n1.0\n1.0\n1.0\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 1.0\n",
    "object": "%%MatrixMarket vector coordinate real general\n2 2 1\n2 1 1.0\n",
    "out_of_bounds": BANNER + "2 2 2\n1 1 1.0\n5 1 2.0\n",
    "zero_index": BANNER + "2 2 1\n0 1 1.0\n",
    "duplicate": BANNER + "2 2 2\n1 1 1.0\n1 1 2.0\n",
    "duplicate_later": BANNER + "3 3 4\n3 3 1\n2 2 1\n3 3 2\n2 2 5\n",
    "trailing_entry": BANNER + "1 1 1\n1 1 1.0\n1 1 extra junk\n",
    "missing_banner": "3 4 3\n1 1 2.5\n",
    "short_banner": "%%MatrixMarket matrix coordinate\n1 1 1\n1 1 1\n",
    "empty": "",
    "only_newline": "\n",
    "no_size": BANNER + "% only comments\n\n",
    "size_missing_nnz": BANNER + "2 2\n",
    "size_trailing": BANNER + "2 2 1 9\n1 1 1\n",
    "size_malformed": BANNER + "2 x 1\n1 1 1\n",
    "zero_dims": BANNER + "0 3 0\n",
    "too_few": BANNER + "3 3 3\n1 1 1\n2 2 2\n",
    "too_few_blank_tail": BANNER + "3 3 3\n1 1 1\n\n2 2 2\n\n",
    "blank_lines_crlf": BANNER.replace("\n", "\r\n") + "2 3 3\r\n\r\n1 3 0.5\r\n  \r\n2 1 -7\r\n2 2 1e-300\r\n\r\n",
    "comment_in_entries": BANNER + "2 2 2\n1 1 1\n% no comments here\n2 2 2\n",
    "missing_value": BANNER + "2 2 1\n1 1\n",
    "missing_column": BANNER + "2 2 1\n1\n",
    "malformed_value": BANNER + "2 2 1\n1 1 1.0x\n",
    "plus_value": BANNER + "2 2 1\n1 1 +1.5\n",
    "plus_index": BANNER + "2 2 1\n+1 1 1.5\n",
    "negative_index": BANNER + "2 2 1\n-1 1 1.5\n",
    "hex_value": BANNER + "2 2 1\n1 1 0x1p3\n",
    "inf_value": BANNER + "2 2 2\n1 1 inf\n2 2 1\n",
    "nan_value": BANNER + "2 2 1\n2 1 nan\n",
    "overflow_value": BANNER + "2 2 1\n1 1 1e999\n",
    "denormal": BANNER + "2 2 2\n1 1 5e-324\n2 2 2.2250738585072014e-308\n",
    "empty_nnz": BANNER + "4 5 0\n",
    "uppercase_banner": "%%MATRIXMARKET MATRIX COORDINATE REAL GENERAL\n2 2 1\n2 2 3.25\n",
    "tabs": BANNER + "2\t2\t2\n1\t2\t0.125\n  2   1    9  \n",
    "unsorted_rows": BANNER + "3 5 6\n3 5 1\n1 4 2\n3 1 3\n1 1 4\n2 3 5\n1 2 6\n",
    "no_final_newline": BANNER + "2 2 1\n2 2 0.75",
    "content_after": BANNER + "1 1 1\n1 1 1.0\n\n\n% trailing comment\n",
}

CSV_CASES = {
    "crlf": "1.5,2\r\n-0.25,4\r\n",
    "ragged": "1,2,3\n4,5\n",
    "empty_cell": "1,,3\n",
    "empty": "",
    "only_newline": "\n",
    "blank_middle": "1,2\n\n3,4\n",
    "spaces": " 1 , 2.5 \n\t3,4\t\n",
    "no_final_newline": "1,2\n3,4",
    "single": "42\n",
    "inf": "1,inf\n",
    "nan": "nan,1\n",
    "malformed": "1,2\n3,4e\n",
    "trailing_comma": "1,2,\n",
    "leading_comma": ",1,2\n",
    "wide_first": "1,2,3\n4,5,6\n7,8\n",
    "cr_only_line": "1,2\n\r\n",
    "exponents": "1e-300,2.5E+10,-0.0\n",
}


def big_mm(seed: int, kind: str) -> str:
    """~2-4 MB Matrix Market text.  kind: 'ok', 'bad_deep' (a malformed value near the
    end), 'dup_deep' (a duplicate pair), 'count' (one entry fewer than declared)."""
    rng = np.random.default_rng(seed)
    m, n = 5003, 4001
    k = 120_000
    flat = rng.choice(m * n, size=k, replace=False)
    rows, cols = flat // n + 1, flat % n + 1
    vals = rng.standard_normal(k) * np.exp(rng.uniform(-20, 20, k))
    lines = [f"{r} {c} {float(v)!r}" for r, c, v in zip(rows, cols, vals)]
    for t in range(0, k, 997):            # sprinkle blank and whitespace-only lines
        lines[t] = lines[t] + "\n" + ("   " if t % 2 else "")
    nnz = k
    if kind == "bad_deep":
        lines[k - 17] = f"{rows[k - 17]} {cols[k - 17]} 1.2.3"
    elif kind == "dup_deep":
        lines[k - 5] = f"{rows[3]} {cols[3]} 9.5"
    elif kind == "count":
        nnz = k + 1
    return BANNER + f"% generated seed {seed}\n{m} {n} {nnz}\n" + "\n".join(lines) + "\n"


def big_csv(seed: int, kind: str) -> str:
    """~2 MB dense CSV; kind 'ok', 'ragged_deep' (a short row near the end), 'bad_deep'."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((2500, 40)) * np.exp(rng.uniform(-30, 30, (2500, 40)))
    lines = [",".join(repr(float(v)) for v in row) for row in x]
    if kind == "ragged_deep":
        lines[2400] = ",".join(repr(float(v)) for v in x[2400, :-1])
    elif kind == "bad_deep":
        lines[2333] = lines[2333].replace(",", ",abc", 1)
    return "\r\n".join(lines) + "\r\n"


BIG_MM = [("big_ok_1", 11, "ok"), ("big_ok_2", 12, "ok"), ("big_bad_deep", 13, "bad_deep"),
          ("big_dup_deep", 14, "dup_deep"), ("big_count", 15, "count")]
BIG_CSV = [("big_ok", 21, "ok"), ("big_ragged_deep", 22, "ragged_deep"), ("big_bad_deep", 23, "bad_deep")]

# values for format_double: the reference test's tricky list (test_data.cpp:105-110) and more
FORMAT_VALUES = [0.1, 1.0 / 3.0, 1e-300, 1e300, 123456789.123456789, 0.0, 5e-324, -0.0, 1.0, 100000.0,
                 1e-5, 1e-4, 0.15000000000000002, 2.0 ** 53, 2.0 ** 53 + 2, 1e15, 1e16, 1e21, 1e22, 123.0,
                 -2.5e-8, 1.7976931348623157e308, 2.2250738585072014e-308, 0.3, 9.999999999999999e22]


def format_values():
    rng = np.random.default_rng(141)
    extra = np.ldexp(rng.uniform(-1, 1, 400), rng.integers(-40, 40, 400))
    return FORMAT_VALUES + [float(v) for v in extra]

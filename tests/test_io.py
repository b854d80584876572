"""Ingestion: the parallel memory-mapped reader against the reference's
open_row_stream (core/src/io.cpp:170-189, compiled from the reference sources) on generated
MatrixMarket and plain files -- row contents, order, empty rows, unsorted entries within a
row, comments, and the error classes. Host-only: runs without a GPU."""
import os

import numpy as np
import pytest

import paper_1602_00412_b200 as P


def _mm(path, rows, d, shuffle_within=True, comments=True, seed=0):
    g = np.random.default_rng(seed)
    nnz = sum(len(r[0]) for r in rows)
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        if comments:
            f.write("% generated\n%\n")
        f.write(f"{len(rows)} {d} {nnz}\n")
        for i, (cs, vs) in enumerate(rows):
            order = g.permutation(len(cs)) if shuffle_within else np.arange(len(cs))
            for k in order:
                f.write(f"{i + 1} {cs[k] + 1} {float(vs[k])!r}\n")
                if comments and k % 7 == 3:
                    f.write("% interleaved comment\n")


def _rows(n, d, density, seed):
    g = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        m = g.random(d) < density
        cs = np.nonzero(m)[0]
        out.append((cs, g.standard_normal(len(cs)) * 10.0 ** g.integers(-3, 4, len(cs))))
    return out


def _check_same(path, reference, plain_cols=0):
    rp, cs, vs, d = P.read_row_stream(path, plain_cols)
    rrp, rcs, rvs, rd, err = reference.read_row_stream(path, plain_cols)
    assert err is None
    assert d == rd and np.array_equal(rp, rrp) and np.array_equal(cs, rcs) and np.array_equal(vs, rvs)
    return rp, cs, vs


@pytest.mark.parametrize("threads", ["1", "3", "16"])
def test_matrix_market_matches_reference(tmp_path, reference, monkeypatch, threads):
    monkeypatch.setenv("SFDG_IO_THREADS", threads)
    rows = _rows(300, 50, 0.08, 1)
    rows[5] = (np.array([], int), np.array([]))  # empty rows inside and at the end
    rows[-1] = (np.array([], int), np.array([]))
    path = str(tmp_path / "a.mtx")
    _mm(path, rows, 50)
    rp, cs, vs = _check_same(path, reference)
    assert len(rp) == 301 and rp[6] == rp[5]


def test_plain_format_matches_reference(tmp_path, reference):
    rows = _rows(200, 40, 0.1, 2)
    path = str(tmp_path / "a.txt")
    with open(path, "w") as f:
        f.write("# plain col:value rows\n")
        for i, (cs, vs) in enumerate(rows):
            if i % 17 == 0:
                f.write("\n   \n")  # blank lines are skipped
            f.write(" ".join(f"{c}:{float(v)!r}" for c, v in zip(cs, vs)) + ("  # tail comment\n" if i % 5 == 0 else "\n"))
    _check_same(path, reference, plain_cols=40)


@pytest.mark.parametrize("body,msg", [
    ("2 3 2\n1 1 1.0\n1 4 2.0\n", "entry index out of range"),
    ("2 3 2\n1 1 1.0\n1 x 2.0\n", "malformed entry line"),
    ("2 3 3\n2 1 1.0\n1 2 2.0\n", "not grouped by nondecreasing row"),
    ("2 3 2\n1 2 1.0\n1 2 2.0\n", "duplicate column within a row"),
    ("x y z\n", "bad MatrixMarket size line"),
])
def test_matrix_market_errors(tmp_path, reference, body, msg):
    path = str(tmp_path / "bad.mtx")
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n" + body)
    with pytest.raises(P.InvalidArgument, match=msg):
        P.read_row_stream(path)
    _, _, _, _, err = reference.read_row_stream(path)
    assert err is not None and msg in err


def test_unsupported_header_and_plain_without_width(tmp_path):
    path = str(tmp_path / "h.mtx")
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix array real general\n2 2\n")
    with pytest.raises(P.InvalidArgument, match="unsupported MatrixMarket header"):
        P.read_row_stream(path)
    path2 = str(tmp_path / "p.txt")
    with open(path2, "w") as f:
        f.write("0:1.0\n")
    with pytest.raises(P.InvalidArgument, match="explicit column count"):
        P.read_row_stream(path2)


def test_large_file_windows(tmp_path, reference, monkeypatch):
    """Rows that straddle the parser's chunk and window boundaries (small SFDG_IO_THREADS
    chunks over a file much larger than a chunk)."""
    monkeypatch.setenv("SFDG_IO_THREADS", "7")
    rows = _rows(2000, 300, 0.05, 3)
    path = str(tmp_path / "big.mtx")
    _mm(path, rows, 300, comments=False)
    _check_same(path, reference)

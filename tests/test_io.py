"""§8(f) row 4: the .tns fast path (include/cpfit_io.h, csrc/io.cpp) against the reference's format
conventions (proj/tests/test_io.cpp:16-83) and against the oracle's sequential restatement of
io.cpp (byte-identical files, identical entries and identical io_error messages), plus the
binary sidecar. CPU only (host code)."""
import os

import numpy as np
import pytest

from conftest import random_sparse


def test_format_double_round_trips(P):
    # test_io.cpp:16-27 with the reference's own Rng(401) stream
    _, uni, _ = P.rng_draws(401, 4000)
    for i in range(2000):
        x = (uni[2 * i] - 0.5) * 10.0 ** (40.0 * (uni[2 * i + 1] - 0.5))
        if i % 7 == 0:
            x = -x
        s = P.format_double(x)
        assert float(s) == x, s
    assert P.format_double(0.0) == "0"
    assert P.format_double(0.1) == "0.1" and P.format_double(1e-7) == "1e-07"


def test_sparse_round_trip_one_based(P, O, tmp_path):
    # test_io.cpp:29-47
    rng = np.random.default_rng(409)
    coords, vals = random_sparse(rng, (3, 4, 2), 0.4)
    path = tmp_path / "t.tns"
    P.write_tns(path, (3, 4, 2), coords, vals)
    text = path.read_text()
    assert text.startswith("tns 3 3 4 ")
    first = text.splitlines()[1].split()
    assert [int(x) for x in first[:3]] == list(coords[0] + 1)
    dims, c2, v2 = P.read_tns(path, sidecar=0)
    assert dims == (3, 4, 2)
    assert np.array_equal(c2, coords) and np.array_equal(v2, vals)
    # the oracle restatement writes the same bytes and reads the same entries
    opath = tmp_path / "o.tns"
    O.tns_write(opath, (3, 4, 2), coords, vals)
    assert opath.read_bytes() == path.read_bytes()
    od, oc, ov = O.tns_read(path)
    assert od == dims and np.array_equal(oc, c2) and np.array_equal(ov, v2)


def test_dense_round_trip(P, tmp_path):
    # test_io.cpp:49-57
    rng = np.random.default_rng(419)
    vals = rng.random(12) * 2 - 1
    path = tmp_path / "d.tns"
    P.write_tns_dense(path, vals, (2, 3, 2))
    dims, back = P.read_tns_dense(path, sidecar=0)
    assert dims == (2, 3, 2) and np.array_equal(back, vals)
    assert path.read_text().splitlines()[0] == "tns 3 2 3 2 12"
    assert path.read_text().splitlines()[2].startswith("2 1 1 ")  # first mode fastest


def test_dense_read_last_duplicate_wins(P, tmp_path):
    # io.cpp:196-200: entries land at their offsets in file order
    path = tmp_path / "dup.tns"
    path.write_text("tns 2 2 2 3\n1 1 1.5\n2 2 4\n1 1 -3\n")
    dims, back = P.read_tns_dense(path, sidecar=0)
    assert np.array_equal(back, [-3.0, 0.0, 0.0, 4.0])


BAD = [
    ("tns 2 2 2 1\n3 1 5.0\n", "bad.tns:2: index out of bounds"),  # test_io.cpp:60-68
    ("tns 2 2 2 2\n1 1 5.0\n", "bad.tns: unexpected end of file, expected tensor entry"),  # truncated
    ("tensor 2 2 2 1\n1 1 5.0\n", "bad.tns:1: expected 'tns' header"),  # wrong magic
    ("tns 2 2 2 1\n1 1 abc\n", "bad.tns:2: expected a number, got 'abc'"),  # bad value
    ("", "bad.tns: unexpected end of file, expected tns header"),
    ("tns 2 2 2\n", "bad.tns:1: tns header needs <N> mode sizes and a count"),
    ("tns x 2 2 1\n", "bad.tns:1: expected an integer, got 'x'"),
    ("tns 2 0 2 1\n1 1 1\n", "bad.tns:1: mode sizes must be >= 1"),
    ("tns 2 2 2 3\n1 1 1\n1 +1 2\n1 2 3\n", "bad.tns:3: expected an integer, got '+1'"),
    ("tns 2 2 2 2\n1 1 1\n\n", "bad.tns:3: entry needs 2 indices and a value"),
    ("tns 2 2 2 2\n1 1 1\n1 1 1 1\n", "bad.tns:3: entry needs 2 indices and a value"),
    ("tns 2 2 2 3\n1 1 1\n2 x 2\n1 2\n", "bad.tns:3: expected an integer, got 'x'"),  # first bad line wins
]


@pytest.mark.parametrize("text,msg", BAD)
def test_diagnostics_name_the_offending_line(P, O, tmp_path, text, msg):
    path = tmp_path / "bad.tns"
    path.write_text(text)
    name = str(path)
    with pytest.raises(P.CpfitIOError) as e:
        P.read_tns(path, sidecar=0)
    assert str(e.value) == msg.replace("bad.tns", name)
    with pytest.raises(O.OracleIOError) as eo:
        O.tns_read(path)
    assert str(eo.value) == str(e.value)


def test_crlf_blank_tail_and_extra_lines(P, O, tmp_path):
    # '\r' dropped (io.cpp:38), tabs and runs of blanks split like istringstream, lines after the
    # nnz-th ignored
    path = tmp_path / "crlf.tns"
    path.write_bytes(b"tns  2 3 2   2\r\n1\t2   0.5\r\n3 1 -2e-3\r\nnot an entry\n")
    dims, c, v = P.read_tns(path, sidecar=0)
    od, oc, ov = O.tns_read(path)
    assert dims == od == (3, 2) and np.array_equal(c, oc) and np.array_equal(v, ov)
    assert np.array_equal(c, [[0, 1], [2, 0]]) and np.array_equal(v, [0.5, -2e-3])


def test_large_file_matches_oracle_and_sidecar(P, O, tmp_path):
    """~600k entries (several thread ranges): product writer bytes == oracle writer bytes; the
    parallel parse == the oracle's sequential parse; the sidecar round trip and its staleness stamp."""
    dims, nnz, R = (300, 200, 100), 600_000, 4
    coords, vals, _ = P.random_sparse_problem(dims, nnz, R, 0.01, 5)
    path, opath = tmp_path / "big.tns", tmp_path / "big_o.tns"
    P.write_tns(path, dims, coords, vals)
    O.tns_write(opath, dims, coords, vals)
    assert path.read_bytes() == opath.read_bytes()
    d, c, v = P.read_tns(path, sidecar=2)  # parse + write <path>.cpfbin
    assert not P.read_tns.last_from_sidecar
    assert os.path.exists(str(path) + ".cpfbin")
    od, oc, ov = O.tns_read(path)
    assert d == od and np.array_equal(c, oc) and np.array_equal(v, ov)
    assert np.array_equal(c, coords) and np.array_equal(v, vals)
    d2, c2, v2 = P.read_tns(path, sidecar=1)
    assert P.read_tns.last_from_sidecar
    assert d2 == d and np.array_equal(c2, c) and np.array_equal(v2, v)
    # a rewritten text file invalidates the sidecar (size / mtime stamp)
    P.write_tns(path, dims, coords[:10], vals[:10])
    d3, c3, v3 = P.read_tns(path, sidecar=1)
    assert not P.read_tns.last_from_sidecar and c3.shape[0] == 10


def test_generators_match_oracle_restatement(P, O):
    """The product's parallel generators (csrc/problems.cpp) against the oracle's sequential
    restatement of problems.cpp (oracle/oracle_problems.cpp): the same draws in the same order;
    starts bit-identical, tensors equal up to the summation order of the noise norms."""
    for dims, R, c, l1, l2 in [((20, 20, 20), 3, 0.5, 1.0, 1.0), ((50, 50, 50), 5, 0.9, 10.0, 5.0),
                               ((12, 10, 8, 6), 4, 0.7, 5.0, 0.0), ((30, 20, 40), 6, 0.5, 1.0, 1.0)]:
        T, truth, _ = P.dense_test_problem(dims, R, c, l1, l2, 0, noise_mode=1, want_truth=True)
        To, tro = O.dense_test_problem(dims, R, c, l1, l2, 0, 1, want_truth=True)
        assert np.abs(T - To).max() <= 1e-14 * np.abs(To).max()
        assert np.abs(truth - tro).max() <= 1e-14
        assert np.array_equal(P.uniform_initial_guess(dims, R, 7), O.uniform_initial_guess(dims, R, 7))
    c1, v1, _ = P.random_sparse_problem((40, 30, 25), 3000, 4, 0.01, 3)
    c2, v2 = O.random_sparse_problem((40, 30, 25), 3000, 4, 0.01, 3)
    assert np.array_equal(c1, c2)
    assert np.abs(v1 - v2).max() <= 1e-14 * np.abs(v2).max()

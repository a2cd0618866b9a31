"""Matrix Market I/O (core/matrix_market.hpp:63-168, synth.hpp:152-168) through
the C ABI: host-only, runs without a GPU. Restates the reference's format and
error behaviour (tests/test_dense_core.cpp's I/O cases)."""
import numpy as np
import pytest

import paper_1012_0365_b200 as B
from paper_1012_0365_b200 import api, synth


def test_dense_roundtrip_bit_exact(tmp_path):
    rs = np.random.default_rng(1)
    a = rs.standard_normal((7, 5)) * 10.0 ** rs.integers(-300, 300, (7, 5))
    p = tmp_path / "a.mtx"
    api.mm_write_dense(p, a)
    lines = p.read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix array real general" and lines[1] == "7 5"
    assert lines[2] == "%.17g" % a[0, 0]  # column-major, 17 significant digits
    assert np.array_equal(api.mm_read_dense(p), a)


def test_sparse_roundtrip_csc(tmp_path):
    m, n = 9, 6
    colptr = np.array([0, 2, 2, 3, 5, 5, 6], dtype=np.int64)
    rowidx = np.array([1, 8, 0, 2, 7, 4], dtype=np.int32)
    vals = np.array([0.1, -2.5, 3.0, 1e-300, 7.0, -0.0])
    p = tmp_path / "s.mtx"
    api.mm_write_sparse(p, m, n, colptr, rowidx, vals)
    text = p.read_text().splitlines()
    assert text[0] == "%%MatrixMarket matrix coordinate real general" and text[1] == "9 6 6"
    assert text[2] == "2 1 0.10000000000000001"  # 1-based, the reference's precision(17)
    r, c, cp, ri, vs = api.mm_read_sparse(p)
    assert (r, c) == (m, n) and np.array_equal(cp, colptr) and np.array_equal(ri, rowidx)
    assert np.array_equal(vs, vals)


def test_reader_sorts_coordinates_and_skips_comments(tmp_path):
    p = tmp_path / "u.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n% a comment\n\n3 2 3\n3 2 1.5\n1 2 2\n2 1 -1\n")
    r, c, cp, ri, vs = api.mm_read_sparse(p)
    assert list(cp) == [0, 1, 3] and list(ri) == [1, 0, 2] and list(vs) == [-1.0, 2.0, 1.5]


@pytest.mark.parametrize("text,kind", [
    ("%%MatrixMarket vector array real general\n1 1\n1\n", "dense"),             # bad banner
    ("%%MatrixMarket matrix array complex general\n1 1\n1\n", "dense"),           # field
    ("%%MatrixMarket matrix array real symmetric\n1 1\n1\n", "dense"),            # symmetry
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n", "dense"),   # format mismatch
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n", "dense"),        # truncated
    ("%%MatrixMarket matrix array real general\n1 1\nnan\n", "dense"),            # non-finite
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n", "sparse"),  # duplicate
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", "sparse"),  # out of range
    ("%%MatrixMarket matrix array real general\n1 1\n1\n", "sparse"),             # format mismatch
    ("", "dense"),                                                                # empty
])
def test_reader_errors(tmp_path, text, kind):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(OSError):
        (api.mm_read_dense if kind == "dense" else api.mm_read_sparse)(p)


def test_missing_file(tmp_path):
    with pytest.raises(OSError):
        api.mm_read_dense(tmp_path / "nope.mtx")


def test_export_instances(tmp_path):
    d, a0, _, _ = synth.rpca_lowrank_sparse(20, 3, 12, 1, B.Rng, B.sample_distinct)
    synth.export_rpca_instance(d, a0, d - a0, tmp_path / "rpca")
    assert np.array_equal(api.mm_read_dense(tmp_path / "rpca" / "d.mtx"), d)
    colptr, rowidx, vals, ml, mr = synth.mc_lowrank(30, 2, 50, 1, B.Rng, B.sample_distinct)
    synth.export_mc_instance(30, 30, colptr, rowidx, vals, ml, mr, tmp_path / "mc")
    r, c, cp, ri, vs = api.mm_read_sparse(tmp_path / "mc" / "observed.mtx")
    assert np.array_equal(cp, colptr) and np.array_equal(ri, rowidx) and np.array_equal(vs, vals)

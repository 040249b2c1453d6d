"""CPU: Matrix Market coordinate I/O (proj/src/matrix_market.cpp:20-142)
against the compiled reference — the same CSR (bit for bit) from the same
file, byte-identical files from the same matrix, the same IoError text for
malformed input."""
import os

import numpy as np
import pytest


def _rand_csr(msc, rng, nr, nc, density):
    a = rng.uniform(-1, 1, (nr, nc)) * (rng.random((nr, nc)) < density)
    a[rng.random((nr, nc)) < 0.02] = 1e-300  # tiny but nonzero
    return msc.SparseMatrix.from_dense(a)


def _same(ours, theirs):
    assert (ours.nrows, ours.ncols) == (theirs.nrows, theirs.ncols)
    assert np.array_equal(ours.row_offsets, theirs.rp)
    assert np.array_equal(ours.col_indices, theirs.ci)
    assert np.array_equal(ours.values.view(np.int64), theirs.v.view(np.int64))


def test_writer_bytes_match_reference(msc, ref, tmp_path):
    rng = np.random.default_rng(7)
    for k, (nr, nc) in enumerate([(1, 1), (17, 9), (40, 40), (3, 120)]):
        a = _rand_csr(msc, rng, nr, nc, 0.3)
        ours, theirs = tmp_path / f"o{k}.mtx", tmp_path / f"r{k}.mtx"
        msc.write_matrix_market(ours, a)
        ref.mm_write(theirs, ref.Csr(a.nrows, a.ncols, *a.arrays()))
        assert ours.read_bytes() == theirs.read_bytes()


def test_reader_matches_reference(msc, ref, tmp_path):
    rng = np.random.default_rng(3)
    # duplicates (summed in the reference's sort order), cancellation to
    # zero, comments / blank lines, symmetric and skew storage, integer field
    cases = []
    lines = ["%%MatrixMarket matrix coordinate real general", "% comment", "", "5 4 9"]
    for _ in range(9):
        lines.append(f"{rng.integers(1, 6)} {rng.integers(1, 5)} {rng.uniform(-1, 1):.17g}")
    cases.append("\n".join(lines) + "\n")
    cases.append("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 0.5\n1 1 -0.5\n"
                 "2 1 0.1\n")
    cases.append("%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 2\n2 1 -1\n"
                 "3 2 -1\n3 3 2\n")
    cases.append("%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 2\n2 1 0.25\n"
                 "3 1 -4\n")
    cases.append("%%MatrixMarket MATRIX Coordinate Integer General\n2 3 2\n1 3 7\n2 2 -1\n")
    for k, text in enumerate(cases):
        p = tmp_path / f"c{k}.mtx"
        p.write_text(text)
        _same(msc.load_matrix_market(p), ref.mm_read(p))


def test_round_trip_cfg1_matrix(msc, ref, tmp_path):
    pb = msc.oseen_problem(32, 0.1, 8)
    C = pb.C
    p = tmp_path / "c.mtx"
    msc.write_matrix_market(p, C)
    back = msc.load_matrix_market(p)
    _same(back, ref.Csr(C.nrows, C.ncols, *C.arrays()))
    _same(back, ref.mm_read(p))


def test_vectors_match_reference(msc, ref, tmp_path):
    v = np.random.default_rng(0).uniform(-1, 1, 50)
    v[::7] = 0.0
    ours, theirs = tmp_path / "o.mtx", tmp_path / "r.mtx"
    msc.write_vector_market(ours, v)
    ref.mm_write_vector(theirs, v)
    assert ours.read_bytes() == theirs.read_bytes()
    assert np.array_equal(msc.load_vector_market(theirs), ref.mm_read_vector(ours))
    assert np.array_equal(msc.load_vector_market(ours), v)


@pytest.mark.parametrize("text", [
    "",
    "%%MatrixMarket vector coordinate real general\n1 1 0\n",
    "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "%%MatrixMarket matrix coordinate real general\n2 x 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 one 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 2\n",
])
def test_errors_match_reference(msc, ref, tmp_path, text):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(ref.RefError) as want:
        ref.mm_read(p)
    with pytest.raises(msc.IoError) as got:
        msc.load_matrix_market(p)
    assert str(got.value) == str(want.value)


def test_missing_file(msc, tmp_path):
    with pytest.raises(msc.IoError, match="cannot open"):
        msc.load_matrix_market(os.path.join(tmp_path, "absent.mtx"))

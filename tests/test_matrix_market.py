"""Matrix Market ingestion: the native reader (sdb_mm_read) against
the reference's own parse of the same files (tests/golden/matrix_market.npz,
tests/golden/mm/*.mtx, made by tests/golden/make_golden.py) and the reference's
contract tests (pkg/tests/test_matrix.py:28-91).  Host code only: no GPU."""

import os

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb

HERE = os.path.dirname(os.path.abspath(__file__))


def _write(path, text):
    path.write_text(text, encoding="ascii")
    return str(path)


def test_reader_matches_reference_parse(golden):
    g = golden("matrix_market")
    for fname in g["files"]:
        mat = sdb.load_matrix_market(os.path.join(HERE, "golden", "mm", str(fname)))
        key = str(fname).replace(".mtx", "")
        np.testing.assert_array_equal(mat.csr.indptr, g[f"{key}_indptr"])
        np.testing.assert_array_equal(mat.csr.indices, g[f"{key}_indices"])
        np.testing.assert_array_equal(mat.csr.data, g[f"{key}_data"])  # bit-exact values
        assert mat.symmetric_storage == bool(g[f"{key}_symmetric_storage"])


def test_load_symmetric_triangle_expands_to_tridiag(tmp_path):
    path = _write(tmp_path / "t.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 5\n1 1 2.0\n2 1 -1.0\n"
                                      "2 2 2.0\n3 2 -1.0\n3 3 2.0\n")
    mat = sdb.load_matrix_market(path)
    np.testing.assert_array_equal(mat.csr.toarray(), [[2.0, -1.0, 0.0], [-1.0, 2.0, -1.0], [0.0, -1.0, 2.0]])


@pytest.mark.parametrize("text,match", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1.0\n2 1 3.0\n", "not symmetric"),
    ("%%MatrixMarket matrix coordinate complex symmetric\n1 1 1\n1 1 1.0 0.0\n", "complex"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n3 1 1.0\n", "out of range"),
    ("%%MatrixMarket matrix array real symmetric\n2 2\n", "format"),
    ("%%MatrixMarket vector coordinate real symmetric\n2 2 0\n", "object"),
    ("%%MatrixMarket matrix coordinate pattern symmetric\n2 2 0\n", "field"),
    ("%%MatrixMarket matrix coordinate real hermitian\n2 2 0\n", "symmetry"),
    ("not a header\n", "missing %%MatrixMarket"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 0\n", "square"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2\n", "size line"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 x\n", "size line"),
    ("%%MatrixMarket matrix coordinate real symmetric\n0 0 0\n", "dimensions"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1\n", "malformed coordinate"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 abc\n", "malformed coordinate"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1.0\n2 2 1.0\n", "more entries"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n", "expected 2 entries, found 1"),
])
def test_reader_errors(tmp_path, text, match):
    with pytest.raises(ValueError, match=match):
        sdb.load_matrix_market(_write(tmp_path / "bad.mtx", text))


def test_load_sums_duplicates_and_empty_list(tmp_path):
    mat = sdb.load_matrix_market(_write(tmp_path / "dup.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
                                                               "2 2 3\n1 1 1.5\n1 1 0.5\n2 1 -1.0\n"))
    np.testing.assert_array_equal(mat.csr.toarray(), [[2.0, -1.0], [-1.0, 0.0]])
    z = sdb.load_matrix_market(_write(tmp_path / "z.mtx", "%%MatrixMarket matrix coordinate real symmetric\n4 4 0\n"))
    assert z.n == 4 and z.csr.nnz == 0


def test_save_load_round_trip_is_exact(tmp_path):
    from paper_1308_5467_b200 import workloads as W

    for op in (W.generate_modified_laplacian_2d(10, 5), sdb.SparseSymmetricMatrix(csr=W.anderson_3d(4).csr)):
        path = tmp_path / "m.mtx"
        sdb.save_matrix_market(op, str(path))
        back = sdb.load_matrix_market(str(path))
        np.testing.assert_array_equal(back.csr.toarray(), op.csr.toarray())
        assert back.symmetric_storage


@pytest.mark.gpu
def test_loaded_matrix_runs_on_device():
    """A file read by the native reader feeds the GPU moment path like any CSR."""
    from oracle import specdens_oracle as O
    from paper_1308_5467_b200 import workloads as W

    mat = sdb.load_matrix_market(os.path.join(HERE, "golden", "mm", "lap20x15.mtx"))
    iv = W.gershgorin_interval(mat)
    src = sdb.ProbeVectorSource("gaussian", seed=0, dim=mat.dim)
    m = sdb.compute_chebyshev_moments(sdb.apply_spectral_map(mat, iv), 40, src, 8)
    ref = O.average_moments(O.chebyshev_moments(mat.csr, iv.center, iv.halfwidth, 40, "gaussian", 0, 8))
    assert np.max(np.abs(m.zeta - ref)) <= 1e-10 * np.max(np.abs(ref))

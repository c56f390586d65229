"""KPM moments and DOS on the GPU: reference contract + parity with the oracle/golden.

The contract tests restate the reference's own pins (pkg/tests/test_kpm.py
:49-178, :290-330) against this package; the parity tests compare the CUDA
path with the reference's golden outputs (tests/golden) and the oracle.
Tolerances: moments max|dz|/max|z| <= 1e-10, DOS max-abs <= 1e-9 (north star).
"""

import numpy as np
import pytest
from numpy.polynomial import chebyshev as npcheb

import paper_1308_5467_b200 as sdb
from oracle import specdens_oracle as O
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.gpu

MOMENT_RTOL = 1e-10
DOS_ATOL = 1e-9
UNIT = sdb.SpectralInterval(-1.0, 1.0)


def basis_source(n):
    return sdb.ProbeVectorSource("basis", seed=0, dim=n)


def unit_operator(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    a = a + a.T
    a *= 0.9 / np.max(np.abs(np.linalg.eigvalsh(a)))
    return sdb.SparseSymmetricMatrix.from_dense(a), np.linalg.eigvalsh(a)


def rel_err(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b))


# ---- reference contract (test_kpm.py) --------------------------------------------


def test_identity_operator_moments_all_ones():
    n = 5
    op = sdb.SparseSymmetricMatrix.from_dense(np.eye(n))
    m = sdb.compute_chebyshev_moments(op, 8, basis_source(n), n_vec=n)
    np.testing.assert_allclose(m.zeta / n, np.ones(9), rtol=0, atol=1e-13)


@pytest.mark.parametrize("fn", [sdb.compute_chebyshev_moments, sdb.moments_via_product_formula])
def test_zero_operator_alternating_pattern(fn):
    n = 4
    op = sdb.SparseSymmetricMatrix.from_dense(np.zeros((n, n)))
    m = fn(op, 6, basis_source(n), n_vec=n)
    np.testing.assert_allclose(m.zeta / n, [1, 0, -1, 0, 1, 0, -1], rtol=0, atol=1e-15)


@pytest.mark.parametrize("fn", [sdb.compute_chebyshev_moments, sdb.moments_via_product_formula])
def test_exhaustive_probes_match_dense_traces(fn):
    op, eigs = unit_operator(12, seed=4)
    m = fn(op, 20, basis_source(12), n_vec=12)
    for k in range(21):
        unit = np.zeros(k + 1)
        unit[k] = 1.0
        assert abs(m.zeta[k] - float(np.sum(npcheb.chebval(eigs, unit)))) <= 1e-10


def test_gaussian_probes_within_error_bars():
    op, eigs = unit_operator(12, seed=4)
    src = sdb.ProbeVectorSource("gaussian", seed=8, dim=12)
    m = sdb.compute_chebyshev_moments(op, 4, src, n_vec=600)  # 3 batches of <= 256
    for k in range(5):
        unit = np.zeros(k + 1)
        unit[k] = 1.0
        assert abs(m.zeta[k] - float(np.sum(npcheb.chebval(eigs, unit)))) <= 4.0 * 12 / np.sqrt(600)


def test_matvec_counts():
    op, _ = unit_operator(10, seed=0)
    counter = sdb.MatvecCounter(op)
    sdb.compute_chebyshev_moments(counter, 17, sdb.ProbeVectorSource("gaussian", 0, 10), n_vec=3)
    assert counter.count == 17 * 3
    for degree in (1, 2, 7, 8, 24):
        counter = sdb.MatvecCounter(op)
        sdb.moments_via_product_formula(counter, degree, sdb.ProbeVectorSource("gaussian", 0, 10), n_vec=3)
        assert counter.count == 3 * ((degree + 1) // 2)


@pytest.mark.parametrize("fn", [sdb.compute_chebyshev_moments, sdb.moments_via_product_formula])
def test_escape_raises_numerical_failure(fn):
    op = sdb.SparseSymmetricMatrix.from_dense(np.diag([3.0]))
    with pytest.raises(sdb.NumericalFailure, match="widen"):
        fn(op, 800, sdb.ProbeVectorSource("gaussian", 0, 1), 1)


def test_truncated_moments_are_exact_prefix():
    op, _ = unit_operator(9, seed=1)
    src = sdb.ProbeVectorSource("gaussian", seed=3, dim=9)
    full = sdb.compute_chebyshev_moments(op, 30, src, n_vec=2)
    short = sdb.compute_chebyshev_moments(op, 12, src, n_vec=2)
    np.testing.assert_array_equal(full.truncated(12).zeta, short.zeta)
    with pytest.raises(ValueError):
        full.truncated(31)


def test_argument_validation():
    op, _ = unit_operator(6, seed=0)
    src = sdb.ProbeVectorSource("gaussian", 0, 6)
    with pytest.raises(ValueError):
        sdb.compute_chebyshev_moments(op, 4, src, 0)
    with pytest.raises(ValueError):
        sdb.compute_chebyshev_moments(op, -1, src, 1)
    with pytest.raises(ValueError, match="stored vectors"):
        sdb.moments_via_product_formula(op, 20, src, n_vec=1, max_stored_vectors=5)
    with pytest.raises(TypeError):

        class MatvecOnly:
            dim = 6

            def matvec(self, x):
                return x

        sdb.compute_chebyshev_moments(MatvecOnly(), 4, src, 1)


def test_degree_zero():
    op, _ = unit_operator(7, seed=2)
    src = sdb.ProbeVectorSource("gaussian", 5, 7)
    for fn in (sdb.compute_chebyshev_moments, sdb.moments_via_product_formula):
        m = fn(op, 0, src, 3)
        ref = np.mean([src.draw(l) @ src.draw(l) for l in range(3)])
        assert m.zeta.shape == (1,) and abs(m.zeta[0] - ref) <= 1e-12 * ref


@pytest.mark.parametrize("degree", list(range(1, 25)))
def test_product_formula_equals_direct(degree):
    op, _ = unit_operator(8, seed=13)
    src = sdb.ProbeVectorSource("gaussian", seed=17, dim=8)
    direct = sdb.compute_chebyshev_moments(op, degree, src, n_vec=2)
    half = sdb.moments_via_product_formula(op, degree, src, n_vec=2)
    assert np.max(np.abs(half.zeta - direct.zeta)) <= 1e-10 * np.max(np.abs(direct.zeta))


def test_jackson_and_coefficients():
    np.testing.assert_allclose(sdb.jackson_damping(1), [1.0, 0.5], rtol=0, atol=1e-15)
    for degree in (1, 5, 50, 200):
        g = sdb.jackson_damping(degree)
        np.testing.assert_allclose(g, O.jackson_damping(degree), rtol=0, atol=1e-14)
        assert np.all(np.diff(g) < 0)
    m = sdb.MomentSequence(zeta=np.full(4, 5.0), degree=3, n_vec=1, basis="chebyshev", n=5)
    np.testing.assert_allclose(sdb.moments_to_coefficients(m, "none"), [1 / np.pi] + [2 / np.pi] * 3, rtol=1e-15)
    m = sdb.MomentSequence(zeta=np.array([1.0, -0.3, 0.2]), degree=2, n_vec=1, basis="chebyshev", n=1)
    np.testing.assert_allclose(sdb.moments_to_coefficients(m, "jackson"),
                               O.moments_to_coefficients(m.zeta, 1, "jackson"), rtol=1e-15, atol=0)


def test_dos_evaluation_contract():
    est = sdb.evaluate_kpm_dos(np.array([1.0 / np.pi]), UNIT, grid=np.array([0.0]))
    assert est.values[0] == pytest.approx(1.0 / np.pi, rel=1e-15)
    with pytest.raises(ValueError, match="1e-06"):
        sdb.evaluate_kpm_dos(np.array([1.0]), UNIT, grid=np.array([1.0]))
    rng = np.random.default_rng(0)
    coeffs = rng.standard_normal(301)
    t = np.linspace(-0.999, 0.999, 777)
    np.testing.assert_allclose(sdb.evaluate_chebyshev_series(coeffs, t), O.evaluate_chebyshev_series(coeffs, t),
                               rtol=0, atol=1e-11)


# ---- parity with the reference's golden outputs ----------------------------------


def _kpm_golden_case(golden, name, matrix):
    g = golden(name)
    iv = sdb.SpectralInterval(float(g["lb"]), float(g["ub"]))
    n_vec, degree, n_pts = int(g["n_vec"]), int(g["degree"]), int(g["n_pts"])
    src = sdb.ProbeVectorSource(str(g["kind"]), seed=0, dim=matrix.dim)
    for pf, zkey, dkey in ((False, "zeta_direct", "estimate_density"),
                           (True, "zeta_product", "estimate_density_product")):
        est = sdb.estimate_dos(matrix, iv, "kpm-jackson", degree, src, n_vec, grid_points=n_pts,
                               product_formula=pf)
        assert rel_err(est.params["moments"], g[zkey]) <= MOMENT_RTOL, (name, pf)
        assert np.max(np.abs(est.density - g[dkey])) <= DOS_ATOL, (name, pf)
        np.testing.assert_array_equal(est.lambda_grid, g["lambda_grid"])
        assert est.params["matvec_count"] == int(g["estimate_matvec_count_product" if pf else "estimate_matvec_count"])
    mapped = sdb.apply_spectral_map(matrix, iv)
    m = sdb.compute_chebyshev_moments(mapped, degree, src, int(g["per_probe_direct"].shape[0]))
    # mean over the first probes equals the mean of the golden per-probe moments
    assert rel_err(m.zeta, g["per_probe_direct"].mean(axis=0)) <= MOMENT_RTOL


def test_golden_c1_full(golden):
    _kpm_golden_case(golden, "c1_kpm", W.build_matrix("C1"))


@pytest.mark.parametrize("auto", ["1", "0"])
def test_golden_c2_subset_stencil_and_csr(golden, monkeypatch, auto):
    monkeypatch.setenv("SDB_AUTO_STENCIL", auto)
    op = W.build_matrix("C2")
    _kpm_golden_case(golden, "c2_subset", op)  # stencil form
    _kpm_golden_case(golden, "c2_subset", sdb.SparseSymmetricMatrix(csr=op.csr))  # CSR (detected or raw)


def test_golden_c3_small(golden):
    _kpm_golden_case(golden, "c3_small", W.dft_like(20000))


@pytest.mark.parametrize("auto", ["1", "0"])
def test_golden_c5_small(golden, monkeypatch, auto):
    monkeypatch.setenv("SDB_AUTO_STENCIL", auto)
    op = W.stencil27_3d(24)
    _kpm_golden_case(golden, "c5_small", op)
    _kpm_golden_case(golden, "c5_small", sdb.SparseSymmetricMatrix(csr=op.csr))


# ---- parity with the oracle on other seeds / shapes ---------------------------------


@pytest.mark.parametrize("n_vec", [1, 2, 3, 12, 20, 32, 64, 100, 128, 200, 256, 300])
def test_oracle_parity_probe_widths(n_vec):
    """Every row-group geometry (L, VPL) against the oracle, both modes."""
    op = W.dft_like(3000, half_band=5, n_random=3)
    iv = W.gershgorin_interval(op)
    degree = 33
    src = sdb.ProbeVectorSource("gaussian", seed=11, dim=op.dim)
    mapped = sdb.apply_spectral_map(op, iv)
    per = O.chebyshev_moments(op, iv.center, iv.halfwidth, degree, "gaussian", 11, n_vec, mode="direct")
    ref = O.average_moments(per)
    got = sdb.compute_chebyshev_moments(mapped, degree, src, n_vec)
    assert rel_err(got.zeta, ref) <= MOMENT_RTOL
    got = sdb.moments_via_product_formula(mapped, degree, src, n_vec)
    assert rel_err(got.zeta, ref) <= MOMENT_RTOL


def test_stencil_equals_csr_form(monkeypatch):
    monkeypatch.setenv("SDB_AUTO_STENCIL", "0")
    op = W.anderson_3d(12)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=1, dim=op.dim)
    a = sdb.moments_via_product_formula(sdb.apply_spectral_map(op, iv), 60, src, 16)
    b = sdb.moments_via_product_formula(sdb.apply_spectral_map(sdb.SparseSymmetricMatrix(csr=op.csr), iv), 60, src,
                                        16)
    assert rel_err(a.zeta, b.zeta) <= 1e-13


def test_deterministic_reruns():
    op = W.anderson_3d(16)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim)
    e1 = sdb.estimate_dos(op, iv, "kpm-jackson", 80, src, 64, grid_points=500, product_formula=True)
    e2 = sdb.estimate_dos(op, iv, "kpm-jackson", 80, src, 64, grid_points=500, product_formula=True)
    np.testing.assert_array_equal(e1.density, e2.density)
    np.testing.assert_array_equal(e1.params["moments"], e2.params["moments"])


def test_csr_stencil_detection():
    from paper_1308_5467_b200.operators import detect_stencil

    for op in (W.anderson_3d(8), W.anderson_3d(12), W.stencil27_3d(6)):
        st = detect_stencil(op.csr)
        assert st is not None and st.shape == op.shape
        np.testing.assert_array_equal(st.diag, op.diag)
        np.testing.assert_array_equal(st.csr.data, op.csr.data)
    assert detect_stencil(W.build_matrix("C1").csr) is None  # Dirichlet faces: not periodic
    assert detect_stencil(W.dft_like(3000, half_band=5, n_random=3).csr) is None
    bad = W.anderson_3d(8).csr.copy()
    bad.data[5] += 1e-3  # one off-diagonal differs: not constant-coefficient
    assert detect_stencil(bad) is None


@pytest.mark.parametrize("shape", ["face7", "box27", "generic"])
def test_stencil_kernels_match_oracle(shape):
    if shape == "face7":
        op = W.anderson_3d(10)
    elif shape == "box27":
        op = W.stencil27_3d(7)
    else:
        rng = np.random.default_rng(1)
        offs = [(1, 0, 0), (-1, 0, 0), (1, 1, 0), (-1, -1, 0), (0, 0, 1), (0, 0, -1)]
        w = [0.3, 0.3, -0.2, -0.2, 0.5, 0.5]
        op = sdb.StencilOperator((5, 6, 7), offs, w, rng.uniform(-1, 1, 210))
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=2, dim=op.dim)
    for n_vec in (1, 20, 32, 64, 130):
        got = sdb.moments_via_product_formula(sdb.apply_spectral_map(op, iv), 41, src, n_vec)
        per = O.chebyshev_moments(op.csr, iv.center, iv.halfwidth, 41, "rademacher", 2, n_vec, mode="direct")
        assert rel_err(got.zeta, O.average_moments(per)) <= MOMENT_RTOL, (shape, n_vec)


@pytest.mark.parametrize("tile", [("8", "2", "1", "1"), ("8", "4", "3", "2"), ("16", "2", "2", "1"),
                                  ("16", "4", "1", "1"), ("8", "2", "0", "3")])
@pytest.mark.parametrize("dims,shape", [((10, 7, 9), "face7"), ((70, 5, 6), "face7"), ((9, 6, 8), "box27"),
                                        ((67, 3, 4), "box27")])
def test_tile_kernel_variants_match_oracle(monkeypatch, tile, dims, shape):
    """2.5-D tile path: slices, tile heights, z segments, partial tiles, nx > 64."""
    cs, ty, zseg, pd = tile
    monkeypatch.setenv("SDB_TILE", "1")
    monkeypatch.setenv("SDB_TILE_PD", pd)
    monkeypatch.setenv("SDB_TILE_CS", cs)
    monkeypatch.setenv("SDB_TILE_TY", ty)
    if zseg != "0":
        monkeypatch.setenv("SDB_TILE_ZSEG", zseg)
    rng = np.random.default_rng(7)
    n = dims[0] * dims[1] * dims[2]
    if shape == "face7":
        offs = W.FACE_OFFSETS
        w = list(rng.uniform(-1, 1, 3).repeat(2))
    else:
        offs, w = [], []
        for o in W._positive_offsets_27():
            v = float(rng.uniform(-1, 1))
            offs += [o, (-o[0], -o[1], -o[2])]
            w += [v, v]
    op = sdb.StencilOperator(dims, offs, w, rng.uniform(-2, 2, n))
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("gaussian", seed=5, dim=n)
    per = O.chebyshev_moments(op.csr, iv.center, iv.halfwidth, 37, "gaussian", 5, 32, mode="direct")
    ref = O.average_moments(per)
    got = sdb.moments_via_product_formula(sdb.apply_spectral_map(op, iv), 37, src, 32)
    assert rel_err(got.zeta, ref) <= MOMENT_RTOL
    grid = sdb.unit_grid(300)
    est = sdb.estimate_dos(op, iv, "kpm-jackson", 37, src, 32, grid_points=300, product_formula=True)
    _, dens = O.evaluate_kpm_dos(O.moments_to_coefficients(ref, n, "jackson"), iv.halfwidth, grid)
    assert np.max(np.abs(est.density - dens)) <= DOS_ATOL


def test_rademacher_sign_staging_is_exact():
    """Sign-bit staging of Rademacher probes gives bit-identical moments to fp64 staging."""

    class PlainSource:  # the reference's protocol only: draw(l) and dim
        def __init__(self, src):
            self.src, self.dim = src, src.dim

        def draw(self, i):
            return self.src.draw(i)

    op = W.anderson_3d(12)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=9, dim=op.dim)
    mapped = sdb.apply_spectral_map(op, iv)
    a = sdb.moments_via_product_formula(mapped, 40, src, 33)
    b = sdb.moments_via_product_formula(mapped, 40, PlainSource(src), 33)
    np.testing.assert_array_equal(a.zeta, b.zeta)


@pytest.mark.parametrize("n_vec", [1, 20, 130])
@pytest.mark.parametrize("pf", [False, True])
def test_csr_with_empty_rows_and_unsorted_entries(n_vec, pf):
    """Rows with no stored entries (zero rows/columns) and rows whose entries are
    not column-sorted: the kernels sum each row in storage order (csr_matvec),
    an empty row contributes -c x / d only."""
    import scipy.sparse as sp

    rng = np.random.default_rng(11)
    n = 500
    a = sp.random(n, n, density=0.01, random_state=3, format="csr")
    a = a + a.T
    dead = rng.choice(n, 60, replace=False)
    keep = np.ones(n)
    keep[dead] = 0.0
    d = sp.diags(keep)
    a = (d @ a @ d).tocsr()
    a.eliminate_zeros()
    assert np.sum(np.diff(a.indptr) == 0) >= 60
    coo = a.tocoo()
    order = rng.permutation(coo.nnz)  # storage order within rows becomes arbitrary
    a = sp.csr_array((coo.data[order], (coo.row[order], coo.col[order])), shape=(n, n))
    a.has_sorted_indices = False
    mat = sdb.SparseSymmetricMatrix(csr=a)
    iv = W.gershgorin_interval(mat)
    src = sdb.ProbeVectorSource("gaussian", seed=5, dim=n)
    fn = sdb.moments_via_product_formula if pf else sdb.compute_chebyshev_moments
    got = fn(sdb.apply_spectral_map(mat, iv), 33, src, n_vec).zeta
    per = O.chebyshev_moments(mat.csr, iv.center, iv.halfwidth, 33, "gaussian", 5, n_vec,
                              mode="product" if pf else "direct")
    assert rel_err(got, O.average_moments(per)) <= MOMENT_RTOL

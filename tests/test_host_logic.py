"""Host-side logic of the drop-in (no GPU): operator-chain resolution, probe
source, argument validation, batching, format detection, config generators."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.operators import detect_stencil, resolve

try:
    import specdens  # the reference, importable only in the build container

    HAVE_REF = True
except Exception:  # pragma: no cover
    HAVE_REF = False


def test_resolve_single_map_and_counters():
    a = sdb.SparseSymmetricMatrix.from_dense(np.diag([1.0, 2.0, 3.0]))
    iv = sdb.SpectralInterval(0.0, 4.0)
    counter = sdb.MatvecCounter(a)
    r = resolve(sdb.apply_spectral_map(counter, iv))
    assert r.base is a and r.c == 2.0 and r.d == 2.0 and r.counters == [counter] and r.dim == 3


def test_resolve_nested_maps_compose():
    rng = np.random.default_rng(0)
    m = rng.standard_normal((6, 6))
    a = sdb.SparseSymmetricMatrix.from_dense(m + m.T)
    inner = sdb.apply_spectral_map(a, sdb.SpectralInterval(-3.0, 5.0))
    outer = sdb.MappedOperator(sdb.MatvecCounter(inner), sdb.SpectralInterval(-0.5, 1.5))
    r = resolve(outer)
    x = rng.standard_normal(6)
    expect = outer.matvec(x)  # host protocol evaluation of the chain
    got = (a.csr @ x - r.c * x) / r.d
    np.testing.assert_allclose(got, expect, rtol=1e-14, atol=1e-14)
    assert len(r.counters) == 1


def test_resolve_accepts_arrays_and_rejects_matvec_only():
    r = resolve(np.eye(3))
    assert r.dim == 3
    r = resolve(sp.csr_array(np.eye(4)))
    assert r.dim == 4

    class MatvecOnly:
        dim = 3

        def matvec(self, x):
            return x

    with pytest.raises(TypeError, match="no CPU fallback"):
        resolve(MatvecOnly())


@pytest.mark.reference
@pytest.mark.skipif(not HAVE_REF, reason="reference not importable")
def test_resolve_reference_objects():
    a = specdens.SparseSymmetricMatrix.from_dense(np.diag([1.0, 2.0]))
    chain = specdens.apply_spectral_map(specdens.MatvecCounter(a), specdens.SpectralInterval(0.0, 4.0))
    r = resolve(chain)
    assert r.base is a and (r.c, r.d) == (2.0, 2.0) and len(r.counters) == 1


@pytest.mark.parametrize("kind", ["gaussian", "rademacher", "basis"])
def test_probe_source_matches_reference_stream(kind):
    src = sdb.ProbeVectorSource(kind, seed=7, dim=50, stream=3)
    blk = src.draw_block(2, 5)
    for i in range(5):
        np.testing.assert_array_equal(np.asarray(blk[i]), src.draw(2 + i))
    if HAVE_REF:
        ref = specdens.ProbeVectorSource(kind, seed=7, dim=50, stream=3)
        for i in range(5):
            np.testing.assert_array_equal(src.draw(i), ref.draw(i))
    with pytest.raises(ValueError):
        sdb.ProbeVectorSource("uniform", 0, 5)


def test_batches_cover_probe_range():
    assert E.batches(600) == [(0, 256), (256, 256), (512, 88)]
    assert E.batches(1) == [(0, 1)]


def test_validation_happens_before_any_device_work():
    a = sdb.SparseSymmetricMatrix.from_dense(np.eye(3))
    src = sdb.ProbeVectorSource("gaussian", 0, 3)
    with pytest.raises(ValueError):
        sdb.compute_chebyshev_moments(a, 4, src, 0)
    with pytest.raises(ValueError):
        sdb.moments_via_product_formula(a, -1, src, 1)
    with pytest.raises(ValueError, match="stored vectors"):
        sdb.moments_via_product_formula(a, 20, src, 1, max_stored_vectors=3)
    with pytest.raises(ValueError, match="sigma"):
        sdb.lanczos_dos(a, sdb.SpectralInterval(0, 2), 2, src, 1, sigma=0.0)
    with pytest.raises(ValueError, match="unknown method"):
        sdb.estimate_dos(a, sdb.SpectralInterval(0, 2), "nope", 4, src, 1)
    with pytest.raises(ValueError, match="product formula"):
        sdb.estimate_dos(a, sdb.SpectralInterval(0, 2), "lanczos", 4, src, 1, sigma=0.1, product_formula=True)
    with pytest.raises(ValueError, match="steps"):
        sdb.estimate_dos(a, sdb.SpectralInterval(0, 2), "cdos", 4, src, 1)
    with pytest.raises(ValueError):
        sdb.lanczos_factorize(a, np.ones(3), 4)
    with pytest.raises(ValueError):
        sdb.lanczos_factorize(a, np.zeros(3), 2)


def test_analytic_counts():
    assert sdb.analytic_matvec_count("kpm", 40, 10) == 400
    assert sdb.analytic_matvec_count("kpm", 40, 10, product_formula=True) == 200
    assert sdb.analytic_matvec_count("spectroscopic", 7, 3, product_formula=True) == 12


def test_value_types():
    iv = sdb.SpectralInterval(-2.0, 6.0)
    assert iv.center == 2.0 and iv.halfwidth == 4.0
    np.testing.assert_allclose(iv.from_unit(iv.to_unit([0.0, 1.0])), [0.0, 1.0])
    with pytest.raises(ValueError):
        sdb.SpectralInterval(1.0, 1.0)
    g = sdb.unit_grid(4)
    np.testing.assert_allclose(g, [-0.75, -0.25, 0.25, 0.75])
    np.testing.assert_allclose(sdb.interval_grid(iv, 2), [0.0, 4.0])
    m = sdb.MomentSequence(zeta=np.arange(5.0), degree=4, n_vec=1, basis="chebyshev", n=3)
    np.testing.assert_array_equal(m.truncated(2).zeta, [0.0, 1.0, 2.0])
    with pytest.raises(ValueError):
        m.truncated(5)


@pytest.mark.reference
@pytest.mark.skipif(not HAVE_REF, reason="reference not importable")
def test_c1_generator_matches_reference_bitwise():
    ref = specdens.generate_modified_laplacian_2d(100, 100, bumps=())
    ours = W.build_matrix("C1")
    for attr in ("indptr", "indices", "data"):
        np.testing.assert_array_equal(getattr(ref.csr, attr), getattr(ours.csr, attr))
    ref = specdens.generate_modified_laplacian_2d(30, 25)
    ours = W.generate_modified_laplacian_2d(30, 25, specdens.DEFAULT_BUMPS)
    np.testing.assert_array_equal(ref.csr.data, ours.csr.data)


def test_workload_shapes():
    c2 = W.build_matrix("C2")
    assert c2.dim == 262144 and c2.nnz == 7 * 262144
    iv = W.gershgorin_interval(c2)
    assert -8.25 <= iv.lambda_lb < -8.2 and 20.2 < iv.lambda_ub <= 20.25
    c5 = W.stencil27_3d(8)
    assert len(c5.offsets) == 26
    for o, w in zip(c5.offsets, c5.weights):  # symmetric weights
        j = c5.offsets.index((-o[0], -o[1], -o[2]))
        assert c5.weights[j] == w
    c3 = W.dft_like(5000)
    assert (c3.csr != c3.csr.T).nnz == 0
    assert 50 < c3.csr.nnz / 5000 < 70


def test_stencil_operator_csr_form_is_exact():
    op = W.anderson_3d(5)
    x = np.random.default_rng(0).standard_normal(op.dim)
    dense = op.csr.toarray()
    np.testing.assert_array_equal(dense, dense.T)
    y = dense @ x
    # independent evaluation of the periodic 7-point stencil
    xx = x.reshape(5, 5, 5)
    ref = (op.diag.reshape(5, 5, 5) * xx
           - sum(np.roll(xx, s, axis=a) for a in range(3) for s in (1, -1))).ravel()
    np.testing.assert_allclose(y, ref, rtol=1e-14, atol=1e-13)


def test_detect_stencil_on_host():
    st = detect_stencil(W.anderson_3d(9).csr)
    assert st is not None and st.shape == (9, 9, 9)
    assert detect_stencil(W.build_matrix("C1").csr) is None


def test_rademacher_sign_bits_round_trip():
    src = sdb.ProbeVectorSource("rademacher", seed=3, dim=1001, stream=2)
    bits = np.asarray(src.draw_block_signs(5, 4))
    assert bits.shape == (4, 126)
    for i in range(4):
        v = np.unpackbits(bits[i], bitorder="little")[:1001] * 2.0 - 1.0
        np.testing.assert_array_equal(v, src.draw(5 + i))
    with pytest.raises(ValueError):
        sdb.ProbeVectorSource("gaussian", 0, 10).draw_block_signs(0, 1)


def test_comparison_validates_before_device_work():
    """pkg/tests/test_compare.py:62-67, :106-112: argument errors come first (no GPU needed)."""
    lap = W.generate_modified_laplacian_2d(10, 5)
    with pytest.raises(ValueError, match="unknown method"):
        sdb.run_method_comparison(lap, ["kpm", "kmp"], [10], sigma=0.4)
    with pytest.raises(ValueError, match="sigma"):
        sdb.run_method_comparison(lap, ["kpm"], [10], sigma=0.0)
    with pytest.raises(ValueError, match="degrees"):
        sdb.run_method_comparison(lap, ["kpm"], [], sigma=0.4)
    with pytest.raises(ValueError, match="degrees"):
        sdb.run_method_comparison(lap, ["kpm"], [0, 10], sigma=0.4)


def test_comparison_golden_rows_are_consistent():
    """The reference's rows in the fixture: exact rows are zero, delta-cheb == kpm, means/std of the errors."""
    import os

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "method_comparison.npz"))
    for name in ("small_lap", "tiny_capped", "basis_full"):
        p = name + "/"
        methods = [str(m) for m in z[p + "row_method"]]
        errs = z[p + "row_errors"]
        np.testing.assert_allclose(errs.mean(axis=1), z[p + "row_mean"], rtol=1e-14)
        np.testing.assert_allclose(errs.std(axis=1, ddof=1), z[p + "row_std"], rtol=1e-12)
        for i, m in enumerate(methods):
            if m == "exact":
                assert np.all(errs[i] == 0.0)
            if m == "delta-cheb":
                j = [k for k, mm in enumerate(methods) if mm == "kpm" and z[p + "row_degree"][k] == z[p + "row_degree"][i]][0]
                np.testing.assert_array_equal(errs[i], errs[j])


@pytest.mark.reference
def test_default_bump_laplacian_matches_reference():
    """generate_modified_laplacian_2d with the default bumps (pkg/src/specdens/matrix.py:173-204)."""
    specdens = pytest.importorskip("specdens")
    ref = specdens.generate_modified_laplacian_2d(12, 9)
    ours = sdb.generate_modified_laplacian_2d(12, 9)
    assert (ref.csr != ours.csr).nnz == 0
    assert sdb.DEFAULT_BUMPS == tuple(tuple(b) for b in specdens.DEFAULT_BUMPS)

"""``run_method_comparison`` on the GPU against the reference's own rows.

The golden file (tests/golden/method_comparison.npz, made by
tests/golden/make_golden_comparison.py from the reference itself) holds every
row the reference returned for two sweeps; the GPU path replays the same calls.
Errors and masses are sup/max-abs densities of O(1e-2): agreement to 1e-9
absolute (the north-star DOS tolerance).  The contract tests of
pkg/tests/test_compare.py:70-112 are restated below.
"""

import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "method_comparison.npz")
TOL = 1e-9


def _case(z, name):
    p = name + "/"
    n = len(z[p + "indptr"]) - 1
    csr = sp.csr_array((z[p + "data"], z[p + "indices"], z[p + "indptr"]), shape=(n, n))
    sigma, eta, n_vec, reps, seed, grid_points, pass_iv = z[p + "scalars"]
    iv = sdb.SpectralInterval(*z[p + "interval"])
    kwargs = dict(eta=None if np.isnan(eta) else float(eta), n_vec=int(n_vec), reps=int(reps), seed=int(seed),
                  probe_kind=str(z[p + "probe_kind"]), grid_points=int(grid_points))
    if pass_iv:
        kwargs.update(interval=iv, spectrum=sdb.ExactSpectrum(eigenvalues=z[p + "eigenvalues"]))
    return sdb.SparseSymmetricMatrix(csr=csr), [str(m) for m in z[p + "methods"]], [int(d) for d in z[p + "degrees"]], \
        float(sigma), kwargs


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["small_lap", "tiny_capped", "basis_full"])
def test_comparison_matches_reference_rows(name):
    z = np.load(GOLDEN)
    mat, methods, degrees, sigma, kwargs = _case(z, name)
    rows = sdb.run_method_comparison(mat, methods, degrees, sigma, **kwargs)
    p = name + "/"
    assert [r.method for r in rows] == [str(m) for m in z[p + "row_method"]]
    assert [r.degree for r in rows] == [int(d) for d in z[p + "row_degree"]]
    assert [r.matvec_count for r in rows] == [int(c) for c in z[p + "row_matvec"]]
    errs = np.stack([r.errors for r in rows])
    np.testing.assert_allclose(errs, z[p + "row_errors"], rtol=0, atol=TOL)
    np.testing.assert_allclose([r.error_mean for r in rows], z[p + "row_mean"], rtol=0, atol=TOL)
    np.testing.assert_allclose([r.error_std for r in rows], z[p + "row_std"], rtol=0, atol=TOL)
    np.testing.assert_allclose([r.mass_mean for r in rows], z[p + "row_mass"], rtol=0, atol=TOL)


@pytest.mark.gpu
def test_dense_eigensolve_and_interval_match_reference():
    z = np.load(GOLDEN)
    mat, *_ = _case(z, "tiny_capped")
    spec = sdb.dense_eigensolve(mat)
    np.testing.assert_allclose(spec.eigenvalues, z["tiny_capped/eigenvalues"], rtol=0, atol=1e-12)
    iv = sdb.estimate_spectral_interval(mat, seed=3)
    np.testing.assert_allclose([iv.lambda_lb, iv.lambda_ub], z["tiny_capped/interval"], rtol=1e-12)


@pytest.mark.gpu
def test_sup_gaussian_of_exact_blur_is_small_and_zero_for_itself():
    mat = W.generate_modified_laplacian_2d(8, 6)
    spec = sdb.dense_eigensolve(mat)
    iv = sdb.spectrum_interval(spec, margin=0.05)
    grid = sdb.interval_grid(iv, 800)
    gauss = sdb.RegularizationKernel("gaussian", 0.4)
    est = sdb.exact_regularized_dos(spec, gauss, grid, iv)
    # phi integrates to ~1 and the metric of the exact blur against itself is the blur-of-blur gap only
    assert est.mass() == pytest.approx(1.0, abs=5e-2)
    rep = sdb.error_sup_gaussian(spec, est, 0.4)
    assert rep.kind == "sup_gaussian" and rep.grid_points == 800 and rep.value > 0
    with pytest.raises(ValueError, match="too coarse"):
        sdb.error_sup_gaussian(spec, est, 0.01)


# pkg/tests/test_compare.py:70-104, restated


@pytest.fixture(scope="module")
def small_lap():
    z = np.load(GOLDEN)
    mat, *_ = _case(z, "small_lap")
    return mat, sdb.SpectralInterval(*z["small_lap/interval"]), sdb.ExactSpectrum(eigenvalues=z["small_lap/eigenvalues"])


@pytest.mark.gpu
def test_comparison_sweep_shares_random_numbers(small_lap):
    mat, iv, spec = small_lap
    rows = sdb.run_method_comparison(mat, ["kpm", "delta-cheb", "exact"], [8, 16], sigma=0.5, n_vec=8, reps=2,
                                     seed=0, grid_points=512, interval=iv, spectrum=spec)
    by_key = {(r.method, r.degree): r for r in rows}
    assert len(rows) == 6
    for deg in (8, 16):
        kpm = by_key[("kpm", deg)]
        dcheb = by_key[("delta-cheb", deg)]
        np.testing.assert_array_equal(kpm.errors, dcheb.errors)
        assert kpm.matvec_count == sdb.analytic_matvec_count("kpm", deg, 8)
        assert len(kpm.errors) == 2
        assert kpm.error_std >= 0.0
    exact = by_key[("exact", 16)]
    assert exact.error_mean == 0.0
    assert exact.matvec_count == 0
    assert exact.mass_mean == pytest.approx(1.0, abs=5e-2)
    assert by_key[("kpm", 16)].mass_mean == pytest.approx(1.0, abs=0.2)


@pytest.mark.gpu
def test_comparison_deduplicates_degrees(small_lap):
    mat, iv, spec = small_lap
    rows = sdb.run_method_comparison(mat, ["lanczos"], [16, 8, 8], sigma=0.5, n_vec=4, reps=1, seed=0,
                                     grid_points=512, interval=iv, spectrum=spec)
    assert [r.degree for r in rows] == [8, 16]
    assert rows[0].error_std == 0.0

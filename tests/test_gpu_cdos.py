"""CDOS on the GPU (lanczos.py:296-368): merge, PCHIP slopes and cell averages in
sdb_cdos_refine, against the reference's own outputs (tests/golden/cdos.npz,
made by tests/golden/make_golden_cdos.py).  Densities max-abs <= 1e-9; the
contract tests of pkg/tests/test_lanczos.py:250-302 are restated.
"""

import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "cdos.npz")
TOL = 1e-9


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN)


def test_cdos_refine_synthetic_matches_reference(z):
    iv = sdb.SpectralInterval(*z["syn/interval"])
    quad = sdb.RitzQuadrature(theta=z["syn/theta"], tau_sq=z["syn/tau"])
    est = sdb.cdos_refine(quad, iv, grid=z["syn/grid"])
    np.testing.assert_allclose(est.params["nodes"], z["syn/nodes"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(est.params["node_weights"], z["syn/node_weights"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(est.density, z["syn/density"], rtol=0, atol=TOL)
    one = sdb.cdos_refine(quad, iv, grid=np.array([0.37]))
    np.testing.assert_allclose(one.density, z["syn/density_one_point"], rtol=0, atol=TOL)
    # the spline helper reproduces the stair midpoints at the nodes
    cdf = est.params["cdf"]
    np.testing.assert_allclose(cdf(cdf.x), cdf.y, atol=1e-14)


def test_cdos_two_node_mass(z):
    quad = sdb.RitzQuadrature(theta=np.array([0.0, 1.0]), tau_sq=np.array([0.5, 0.5]))
    interval = sdb.SpectralInterval(-0.5, 1.5)
    grid = sdb.interval_grid(interval, 4001)
    est = sdb.cdos_refine(quad, interval, grid=grid)
    np.testing.assert_allclose(est.density, z["two/density"], rtol=0, atol=TOL)
    assert est.density.sum() * (grid[1] - grid[0]) == pytest.approx(1.0, abs=1e-12)
    assert np.trapezoid(est.density, grid) == pytest.approx(1.0, abs=1e-3)
    assert np.all(est.density >= 0.0)


def test_cdos_dos_matches_reference(z):
    n = len(z["lap/indptr"]) - 1
    lap = sdb.SparseSymmetricMatrix(csr=sp.csr_array((z["lap/data"], z["lap/indices"], z["lap/indptr"]), shape=(n, n)))
    iv = sdb.SpectralInterval(*z["lap/interval"])
    grid = sdb.interval_grid(iv, 512)
    est = sdb.cdos_dos(lap, iv, 20, sdb.ProbeVectorSource("gaussian", seed=3, dim=n), 8, grid=grid)
    np.testing.assert_allclose(est.params["ritz_nodes"], z["lap/ritz_nodes"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(est.params["ritz_weights"], z["lap/ritz_weights"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(est.density, z["lap/density"], rtol=0, atol=TOL * max(1.0, z["lap/density"].max()))


def test_estimate_dos_cdos_matches_reference(z):
    op = W.anderson_3d(8)
    iv = sdb.SpectralInterval(*z["and/interval"])
    est = sdb.estimate_dos(op, iv, "cdos", 30, sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim), 6,
                           grid_points=300)
    np.testing.assert_array_equal(est.lambda_grid, z["and/lambda_grid"])
    np.testing.assert_allclose(est.density, z["and/density"], rtol=0, atol=TOL * max(1.0, z["and/density"].max()))
    assert est.params["matvec_count"] == int(z["and/matvec_count"])
    assert est.method == "cdos"


def test_cdos_full_run_matches_staircase_counts():
    lam = np.array([0.5, 1.1, 2.0, 3.3, 4.1, 5.0])
    n = len(lam)
    op = sdb.SparseSymmetricMatrix.from_dense(np.diag(lam))
    interval = sdb.SpectralInterval(0.0, 5.5)
    grid = sdb.interval_grid(interval, 2201)
    est = sdb.cdos_dos(op, interval, n, sdb.ProbeVectorSource("basis", seed=0, dim=n), n, grid=grid)
    from scipy.integrate import cumulative_trapezoid

    cdf = cumulative_trapezoid(est.density, grid, initial=0.0)
    for k, lam_k in enumerate(lam, start=1):
        value = np.interp(lam_k, grid, cdf)
        assert abs(value - (k / n - 1.0 / (2 * n))) <= 1.2 / (2 * n)


def test_cdos_needs_two_nodes():
    quad = sdb.RitzQuadrature(theta=np.array([1.0]), tau_sq=np.array([1.0]))
    with pytest.raises(ValueError, match="Ritz nodes"):
        sdb.cdos_refine(quad, sdb.SpectralInterval(0.0, 2.0))

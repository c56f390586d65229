"""Hutchinson trace estimation and the heat-capacity functional on the GPU, against
the reference's own outputs (tests/golden/extras.npz, made by
tests/golden/make_golden_extras.py), plus pkg/tests/test_stochastic.py:60-99
restated for the device path.
"""

import os

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "extras.npz")


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN)


def test_trace_matches_reference(z):
    lap = W.build_matrix("C1")
    t = sdb.estimate_trace_quadratic(lap, sdb.ProbeVectorSource("gaussian", seed=0, dim=lap.dim), 50)
    v, n, var = z["trace/c1"]
    assert t.n_samples == int(n)
    assert t.value == pytest.approx(v, rel=1e-12)
    assert t.sample_variance == pytest.approx(var, rel=1e-10)
    op = W.anderson_3d(8)
    t = sdb.estimate_trace_quadratic(op, sdb.ProbeVectorSource("rademacher", seed=1, dim=op.dim), 20)
    v, n, var = z["trace/and8"]
    assert t.value == pytest.approx(v, rel=1e-12)
    assert t.sample_variance == pytest.approx(var, rel=1e-10)


def test_trace_diag_rademacher_is_exact_with_zero_variance():
    d = np.array([1.0, -2.0, 3.5, 0.25])
    mat = sdb.SparseSymmetricMatrix.from_dense(np.diag(d))
    counter = sdb.MatvecCounter(mat)
    est = sdb.estimate_trace_quadratic(counter, sdb.ProbeVectorSource("rademacher", seed=2, dim=4), n_vec=8)
    assert est.value == pytest.approx(d.sum(), abs=1e-14)
    assert est.sample_variance == pytest.approx(0.0, abs=1e-24)
    assert counter.count == 8


def test_trace_of_identity_gaussian_within_error_bars():
    eye = sdb.SparseSymmetricMatrix.from_dense(np.eye(50))
    est = sdb.estimate_trace_quadratic(eye, sdb.ProbeVectorSource("gaussian", seed=0, dim=50), n_vec=400)
    assert abs(est.value - 50.0) <= 4.0 * np.sqrt(est.sample_variance / 400)


def test_heat_capacity_matches_reference(z):
    temps = z["heat/temps"]
    np.testing.assert_allclose(sdb.default_temperatures(), temps, rtol=0, atol=0)
    spec = sdb.ExactSpectrum(eigenvalues=z["heat/eigs"])
    np.testing.assert_allclose(sdb.heat_capacity(spec, temps), z["heat/exact"], rtol=1e-12, atol=1e-14)
    iv = sdb.SpectralInterval(*z["heat/interval"])
    est = sdb.SpectralDensityEstimate.from_original(z["heat/grid"], z["heat/density"], iv, method="exact")
    np.testing.assert_allclose(sdb.heat_capacity(est, temps), z["heat/estimate"], rtol=1e-12, atol=1e-14)
    quad = sdb.RitzQuadrature(theta=z["heat/theta"], tau_sq=z["heat/tau"])
    np.testing.assert_allclose(sdb.heat_capacity(quad, temps, normalize=False), z["heat/ritz"], rtol=1e-12,
                               atol=1e-14)
    with pytest.raises(ValueError, match="temperatures"):
        sdb.heat_capacity(spec, [0.0, 1.0])
    with pytest.raises(ValueError, match="negative"):
        sdb.heat_capacity(sdb.ExactSpectrum(eigenvalues=np.array([-1.0, 1.0])), temps)

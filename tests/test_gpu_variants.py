"""Moment-sharing variants on the GPU: Legendre moments from the
fused step kernels, KPML, spectroscopic and delta-Chebyshev densities.

Reference contract tests restated from pkg/tests/test_kpm.py:184-207, parity
against the reference's own outputs (tests/golden/variants_*.npz, made by
tests/golden/make_golden.py).  Tolerances: moments max|dz|/max|z| <= 1e-10,
densities max-abs <= 1e-9.
"""

import numpy as np
import pytest
from numpy.polynomial import legendre as npleg

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import _native
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.operators import device_matrix, resolve

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


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b))


# ---- reference contract (test_kpm.py:184-207) ------------------------------------


def test_legendre_moments_identity_operator():
    n = 5
    op = sdb.SparseSymmetricMatrix.from_dense(np.eye(n))
    m = sdb.compute_legendre_moments(op, 8, basis_source(n), n_vec=n)
    assert m.basis == "legendre"
    np.testing.assert_allclose(m.zeta / n, np.ones(9), rtol=0, atol=1e-13)


def test_legendre_moments_zero_operator():
    n = 4
    op = sdb.SparseSymmetricMatrix.from_dense(np.zeros((n, n)))
    m = sdb.compute_legendre_moments(op, 4, basis_source(n), n_vec=n)
    np.testing.assert_allclose(m.zeta / n, [1.0, 0.0, -0.5, 0.0, 0.375], rtol=0, atol=1e-15)


def test_legendre_moments_match_dense_trace_oracle():
    op, eigs = unit_operator(12, seed=6)
    m = sdb.compute_legendre_moments(op, 18, basis_source(12), n_vec=12)
    for k in range(19):
        unit = np.zeros(k + 1)
        unit[k] = 1.0
        assert abs(m.zeta[k] - float(np.sum(npleg.legval(eigs, unit)))) <= 1e-10


def test_legendre_matvec_count_and_errors():
    op, _ = unit_operator(10, seed=0)
    counter = sdb.MatvecCounter(op)
    sdb.compute_legendre_moments(counter, 13, sdb.ProbeVectorSource("gaussian", 0, 10), n_vec=3)
    assert counter.count == 13 * 3
    with pytest.raises(ValueError):
        sdb.compute_legendre_moments(op, 4, sdb.ProbeVectorSource("gaussian", 0, 10), 0)
    m = sdb.MomentSequence(zeta=np.ones(3), degree=2, n_vec=1, basis="chebyshev", n=1)
    with pytest.raises(ValueError):
        sdb.evaluate_kpml_dos(m, UNIT)
    leg = sdb.MomentSequence(zeta=np.ones(3), degree=2, n_vec=1, basis="legendre", n=1)
    with pytest.raises(ValueError):
        sdb.moments_to_coefficients(leg)
    with pytest.raises(ValueError, match="1e-06"):
        sdb.evaluate_kpml_dos(leg, UNIT, grid=np.array([1.0]))


def test_legendre_series_matches_numpy():
    rng = np.random.default_rng(1)
    c = rng.standard_normal(257)
    t = np.linspace(-0.999, 0.999, 501)
    np.testing.assert_allclose(sdb.evaluate_legendre_series(c, t), npleg.legval(t, c), rtol=0, atol=1e-10)
    np.testing.assert_allclose(sdb.evaluate_legendre_series(c[:1], t), np.full_like(t, c[0]), rtol=0, atol=0)


def test_delta_cheb_uniform_equals_undamped_kpm():
    op, _ = unit_operator(10, seed=3)
    src = sdb.ProbeVectorSource("gaussian", 2, 10)
    m = sdb.compute_chebyshev_moments(op, 30, src, 4)
    grid = sdb.unit_grid(64)
    kpm = sdb.evaluate_kpm_dos(sdb.moments_to_coefficients(m), UNIT, grid)
    delta = sdb.delta_chebyshev_dos(m, UNIT, grid)
    np.testing.assert_array_equal(kpm.density, delta.density)
    with pytest.raises(ValueError):
        sdb.delta_chebyshev_dos(m, UNIT, grid, degrees=np.full(64, 31))


# ---- parity with the reference's outputs ------------------------------------------


def _variants(golden, name, op):
    g = golden(name)
    iv = sdb.SpectralInterval(float(g["lb"]), float(g["ub"]))
    n_vec, degree, n_pts = int(g["n_vec"]), int(g["degree"]), int(g["n_pts"])
    src = sdb.ProbeVectorSource(str(g["kind"]), seed=0, dim=op.dim)
    mapped = sdb.apply_spectral_map(op, iv)
    grid = sdb.unit_grid(n_pts)
    leg = sdb.compute_legendre_moments(mapped, degree, src, n_vec)
    assert rel(leg.zeta, g["zeta_legendre"]) <= MOMENT_RTOL
    kpml = sdb.evaluate_kpml_dos(leg, iv, grid)
    assert np.max(np.abs(kpml.density - g["kpml_density"])) <= DOS_ATOL
    cheb = sdb.compute_chebyshev_moments(mapped, degree, src, n_vec)
    assert rel(cheb.zeta, g["zeta_chebyshev"]) <= MOMENT_RTOL
    assert np.max(np.abs(sdb.spectroscopic_dos(cheb, iv, grid).density - g["spectroscopic_density"])) <= DOS_ATOL
    delta = sdb.delta_chebyshev_dos(cheb, iv, grid, degrees=g["delta_degrees"])
    assert np.max(np.abs(delta.density - g["delta_density"])) <= DOS_ATOL
    for method in ("kpml", "spectroscopic", "delta-cheb"):
        est = sdb.estimate_dos(op, iv, method, degree, src, n_vec, grid_points=n_pts)
        assert np.max(np.abs(est.density - g[f"estimate_{method}_density"])) <= DOS_ATOL, method
        assert est.params["matvec_count"] == int(g[f"estimate_{method}_matvec_count"])
    # Delta-Gauss-Legendre on the same Legendre moments (dgl.py:109-132)
    sigma = float(g["dgl_sigma"])
    dgl = sdb.evaluate_dgl_dos(leg, iv, sigma, grid)
    assert np.max(np.abs(dgl.density - g["dgl_density"])) <= DOS_ATOL
    assert dgl.params["effective_degree"] == int(g["dgl_effective_degree"])
    est = sdb.estimate_dos(op, iv, "dgl", degree, src, n_vec, sigma=sigma, grid_points=n_pts)
    assert np.max(np.abs(est.density - g["estimate_dgl_density"])) <= DOS_ATOL
    assert est.params["matvec_count"] == int(g["estimate_dgl_matvec_count"])
    for i in range(4):
        co = sdb.compute_dgl_coefficients(float(g[f"dglcoef{i}_t"]), 0.05, degree)
        assert co.effective_degree == int(g[f"dglcoef{i}_effective"])
        np.testing.assert_allclose(co.gamma, g[f"dglcoef{i}_gamma"], rtol=0, atol=1e-12)
        psi_ref = g[f"dglcoef{i}_psi"]
        # psi is a running sum of an unstable recurrence: erf/exp ulps grow towards the cutoff
        assert np.max(np.abs(co.psi - psi_ref)) <= 1e-10 * np.max(np.abs(psi_ref))


def test_variants_c1_csr(golden):
    _variants(golden, "variants_c1", W.build_matrix("C1"))


@pytest.mark.parametrize("zmarch", ["1", "0"])
def test_variants_c5small_stencil_kernels(golden, monkeypatch, zmarch):
    """27-point stencil, 32 probes: the TMA z-march kernel and the row-panel grid
    kernel both run the Legendre update."""
    monkeypatch.setenv("SDB_ZMARCH", zmarch)
    op = W.stencil27_3d(24)
    dm = device_matrix(resolve(op).base, 0, E.stream_ptr(0))
    name = _native.load().sdb_cheb_kernel(dm.handle, 32, _native.SDB_LEGENDRE).decode()
    assert name == ("cheb_step_zmarch" if zmarch == "1" else "cheb_step_grid")
    _variants(golden, "variants_c5small", op)
    # the CSR form of the same operator (stencil detection off -> CSR kernel)
    monkeypatch.setenv("SDB_AUTO_STENCIL", "0")
    _variants(golden, "variants_c5small", sdb.SparseSymmetricMatrix(csr=op.csr))


def test_dgl_contract():
    """dgl.py contract: argument checks, gamma_0 closed form, kernel halting."""
    with pytest.raises(ValueError):
        sdb.compute_dgl_coefficients(1.0, 0.1, 10)
    with pytest.raises(ValueError):
        sdb.compute_dgl_coefficients(0.0, 0.0, 10)
    with pytest.raises(ValueError):
        sdb.compute_dgl_coefficients(0.0, 0.1, 10, tol=0.0)
    co = sdb.compute_dgl_coefficients(0.2, 0.1, 200)
    assert co.gamma[0] == pytest.approx(float(sdb.gamma_zero(0.2, 0.1)), rel=1e-14)
    assert 1 <= co.effective_degree <= 200 and len(co.gamma) == co.effective_degree + 1
    m = sdb.MomentSequence(zeta=np.ones(3), degree=2, n_vec=1, basis="chebyshev", n=1)
    with pytest.raises(ValueError):
        sdb.evaluate_dgl_dos(m, UNIT, 0.1)
    leg = sdb.MomentSequence(zeta=np.ones(3), degree=2, n_vec=1, basis="legendre", n=1)
    with pytest.raises(ValueError):
        sdb.evaluate_dgl_dos(leg, UNIT, 0.1, grid=np.array([1.0]))
    with pytest.raises(ValueError):
        sdb.evaluate_dgl_dos(leg, UNIT, -0.1)

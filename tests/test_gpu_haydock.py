"""Haydock resolvent DOS on the GPU: the batched Lanczos
tridiagonals stay on the device; one kernel evaluates each probe's continued
fraction and the Thomas truncation diagnostic per grid point.

Contract tests restated from pkg/tests/test_lanczos.py:207-247 and
test_acceptance.py:199-224; parity with the reference's outputs
(tests/golden/haydock_*.npz).  Densities max-abs <= 1e-9 (relative to the
peak density); resolvents <= 1e-10.
"""

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.gpu


def random_symmetric(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    a = 0.5 * (a + a.T)
    return sdb.SparseSymmetricMatrix.from_dense(a), a


def test_haydock_single_site_is_lorentzian():
    op = sdb.SparseSymmetricMatrix.from_dense(np.array([[0.4]]))
    iv = sdb.SpectralInterval(-1.0, 1.0)
    grid = sdb.interval_grid(iv, 157)
    est = sdb.haydock_dos(op, iv, 1, sdb.ProbeVectorSource("gaussian", seed=1, dim=1), 1, eta=0.2, grid=grid)
    lorentz = 0.2 / np.pi / ((grid - 0.4) ** 2 + 0.2**2)
    np.testing.assert_allclose(est.density, lorentz, rtol=1e-12)


def test_continued_fraction_two_level_value():
    val = sdb.continued_fraction_resolvent(np.zeros(2), np.ones(1), np.array([2.0 + 0.0j]))
    assert val[0] == pytest.approx(2.0 / 3.0, abs=1e-15)


@pytest.mark.parametrize("n,m", [(16, 10), (120, 100)])
def test_resolvent_routes_agree(n, m):
    """Continued fraction == Thomas solve == Ritz pole sum (acceptance criterion 6)."""
    op, a = random_symmetric(n, 23 + n)
    rng = np.random.default_rng(6)
    fact = sdb.lanczos_factorize(op, rng.standard_normal(n), m)
    quad = sdb.ritz_quadrature(fact)
    lam = np.linalg.eigvalsh(a)
    worst = 0.0
    for eta in (0.05, 0.1, 0.35):
        z = np.linspace(lam[0] - 1.0, lam[-1] + 1.0, 200) + 1j * eta
        cf = sdb.continued_fraction_resolvent(fact.alpha, fact.beta, z)
        th, _ = sdb.tridiagonal_resolvent_first(fact.alpha, fact.beta, z)
        poles = np.sum(quad.tau_sq[:, None] / (z[None, :] - quad.theta[:, None]), axis=0)
        worst = max(worst, float(np.max(np.abs(cf - th))), float(np.max(np.abs(cf - poles))))
    assert worst <= 1e-10


def test_haydock_defaults_and_diagnostics():
    op, a = random_symmetric(12, 31)
    lam = np.linalg.eigvalsh(a)
    iv = sdb.SpectralInterval(lam[0] - 0.3, lam[-1] + 0.3)
    grid = sdb.interval_grid(iv, 256)
    est = sdb.haydock_dos(op, iv, 8, sdb.ProbeVectorSource("rademacher", seed=2, dim=12), 3, grid=grid)
    assert est.params["eta"] == pytest.approx(iv.width / 512.0)
    assert est.params["truncation_indicator"] >= 0.0
    assert np.all(est.density >= 0.0)
    with pytest.raises(ValueError):
        sdb.haydock_dos(op, iv, 8, sdb.ProbeVectorSource("rademacher", seed=2, dim=12), 3, eta=0.0, grid=grid)


@pytest.mark.parametrize("name,build", [("haydock_small", lambda: W.anderson_3d(8)),
                                        ("haydock_c4", lambda: W.build_matrix("C4"))])
def test_haydock_matches_reference(golden, name, build):
    g = golden(name)
    op = build()
    iv = sdb.SpectralInterval(float(g["lb"]), float(g["ub"]))
    src = sdb.ProbeVectorSource(str(g["kind"]), seed=0, dim=op.dim)
    steps, n_vec, eta = int(g["steps"]), int(g["n_vec"]), float(g["eta"])
    grid = g["grid"]
    scale = float(np.max(g["density"]))
    est = sdb.haydock_dos(op, iv, steps, src, n_vec, eta=eta, grid=grid)
    assert np.max(np.abs(est.density - g["density"])) <= 1e-9 * scale
    assert abs(est.params["truncation_indicator"] - float(g["trunc"])) <= 1e-6 * max(float(g["trunc"]), 1e-300) + 1e-12
    est_d = sdb.haydock_dos(op, iv, steps, src, n_vec, grid=grid)
    assert est_d.params["eta"] == float(g["default_eta"])
    assert np.max(np.abs(est_d.density - g["density_default_eta"])) <= 1e-9 * float(np.max(g["density_default_eta"]))
    est2 = sdb.estimate_dos(op, iv, "haydock", steps, src, n_vec, eta=eta, grid_points=int(g["n_pts"]))
    assert np.max(np.abs(est2.density - g["estimate_density"])) <= 1e-9 * scale
    assert est2.params["matvec_count"] == int(g["estimate_matvec_count"])
    cf = sdb.continued_fraction_resolvent(g["alpha0"], g["beta0"], g["z"])
    assert np.max(np.abs(cf - g["cf"])) <= 1e-12 * np.max(np.abs(g["cf"]))
    w0, wl = sdb.tridiagonal_resolvent_first(g["alpha0"], g["beta0"], g["z"])
    assert np.max(np.abs(w0 - g["w_first"])) <= 1e-12 * np.max(np.abs(g["w_first"]))
    assert np.max(np.abs(wl - g["w_last"])) <= 1e-10 * np.max(np.abs(g["w_last"]))

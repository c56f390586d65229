"""Pin the CPU oracle against the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py from /root/reference).  No GPU needed."""

import hashlib

import numpy as np
import pytest

from oracle import specdens_oracle as O
from paper_1308_5467_b200 import workloads as W


def csr_digest(csr):
    h = hashlib.sha256()
    for a in (csr.indptr.astype(np.int64), csr.indices.astype(np.int64), csr.data.astype(np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


KPM_CASES = {
    "c1_kpm": lambda: W.build_matrix("C1"),
    "c3_small": lambda: W.dft_like(20000),
    "c5_small": lambda: W.stencil27_3d(24),
    "c2_subset": lambda: W.build_matrix("C2"),
}


@pytest.mark.parametrize("name", list(KPM_CASES))
def test_generators_match_fixture_matrix(golden, name):
    g = golden(name)
    op = KPM_CASES[name]()
    assert csr_digest(op.csr) == str(g["matrix_sha256"])
    iv = W.gershgorin_interval(op)
    assert (iv.lambda_lb, iv.lambda_ub) == (float(g["lb"]), float(g["ub"]))


@pytest.mark.parametrize("name", ["c1_kpm", "c3_small", "c5_small", "c2_subset"])
def test_oracle_moments_match_reference(golden, name):
    g = golden(name)
    op = KPM_CASES[name]()
    c = 0.5 * (float(g["lb"]) + float(g["ub"]))
    d = 0.5 * (float(g["ub"]) - float(g["lb"]))
    n_vec, degree = int(g["n_vec"]), int(g["degree"])
    per = O.chebyshev_moments(op.csr, c, d, degree, str(g["kind"]), 0, n_vec, mode="direct")
    zeta = O.average_moments(per)
    # same arithmetic as the reference: bit-for-bit
    np.testing.assert_array_equal(zeta, g["zeta_direct"])
    np.testing.assert_array_equal(per[: g["per_probe_direct"].shape[0]], g["per_probe_direct"])
    perp = O.chebyshev_moments(op.csr, c, d, degree, str(g["kind"]), 0, n_vec, mode="product")
    np.testing.assert_array_equal(O.average_moments(perp), g["zeta_product"])
    # the doubling identities the GPU kernel uses agree to ~1e-13
    perd = O.chebyshev_moments(op.csr, c, d, degree, str(g["kind"]), 0, n_vec, mode="doubling")
    zd = O.average_moments(perd)
    assert np.max(np.abs(zd - zeta)) / np.max(np.abs(zeta)) <= 1e-12
    # DOS
    t = O.unit_grid(int(g["n_pts"]))
    values, density = O.evaluate_kpm_dos(O.moments_to_coefficients(zeta, op.dim, "jackson"), d, t)
    np.testing.assert_array_equal(values, g["values_direct"])
    np.testing.assert_array_equal(density, g["density_direct"])
    np.testing.assert_array_equal(density, g["estimate_density"])
    assert int(g["estimate_matvec_count"]) == n_vec * degree
    assert int(g["estimate_matvec_count_product"]) == n_vec * ((degree + 1) // 2)


@pytest.mark.parametrize("name,builder", [("lanczos_small", lambda: W.anderson_3d(8)),
                                          ("c4_subset", lambda: W.build_matrix("C4"))])
def test_oracle_lanczos_matches_reference(golden, name, builder):
    g = golden(name)
    op = builder()
    assert csr_digest(op.csr) == str(g["matrix_sha256"])
    n_vec = int(g["n_vec"]) if name == "lanczos_small" else 1
    dens, theta, tau, facts = O.lanczos_dos(op.csr, int(g["steps"]), str(g["kind"]), 0, n_vec, float(g["sigma"]),
                                            g["grid"])
    for l, (a, b, bn) in enumerate(facts[: g["alpha"].shape[0]]):
        np.testing.assert_array_equal(a, g["alpha"][l])
        np.testing.assert_array_equal(b, g["beta"][l])
        assert bn == g["beta_next"][l]
    if name == "lanczos_small":
        np.testing.assert_array_equal(theta, g["ritz_nodes"])
        np.testing.assert_array_equal(tau, g["ritz_weights"])
        np.testing.assert_allclose(dens, g["density"], rtol=0, atol=1e-15)


def test_oracle_small_contracts():
    # zero operator with exhaustive probes: 1, 0, -1, 0, ...
    z = np.zeros((4, 4))
    per = O.chebyshev_moments(z, 0.0, 1.0, 6, "basis", 0, 4)
    np.testing.assert_allclose(O.average_moments(per) / 4, [1, 0, -1, 0, 1, 0, -1], atol=1e-15)
    np.testing.assert_allclose(O.jackson_damping(1), [1.0, 0.5], atol=1e-15)
    with pytest.raises(ValueError):
        O.evaluate_kpm_dos(np.array([1.0]), 1.0, np.array([1.0]))
    with pytest.raises(O.OracleNumericalFailure):
        O.average_moments(O.chebyshev_moments(np.diag([3.0]), 0.0, 1.0, 800, "gaussian", 0, 1))


VARIANT_CASES = {"variants_c1": lambda: W.build_matrix("C1"), "variants_c5small": lambda: W.stencil27_3d(24)}


@pytest.mark.parametrize("name", list(VARIANT_CASES))
def test_oracle_variants_match_reference(golden, name):
    """Legendre moments, KPML, spectroscopic and delta-Chebyshev (kpm.py:110-124, :220-308)."""
    g = golden(name)
    op = VARIANT_CASES[name]()
    assert csr_digest(op.csr) == str(g["matrix_sha256"])
    lb, ub = float(g["lb"]), float(g["ub"])
    c, d = 0.5 * (lb + ub), 0.5 * (ub - lb)
    n_vec, degree, n = int(g["n_vec"]), int(g["degree"]), int(g["n"])
    t = O.unit_grid(int(g["n_pts"]))
    leg = O.average_moments(O.chebyshev_moments(op.csr, c, d, degree, str(g["kind"]), 0, n_vec, mode="legendre"))
    np.testing.assert_array_equal(leg, g["zeta_legendre"])
    vals, dens = O.kpml_dos(leg, n, d, t)
    np.testing.assert_array_equal(vals, g["kpml_values"])
    np.testing.assert_array_equal(dens, g["kpml_density"])
    cheb = O.average_moments(O.chebyshev_moments(op.csr, c, d, degree, str(g["kind"]), 0, n_vec))
    np.testing.assert_array_equal(cheb, g["zeta_chebyshev"])
    np.testing.assert_array_equal(O.spectroscopic_dos(cheb, n, d, t)[1], g["spectroscopic_density"])
    np.testing.assert_array_equal(O.delta_chebyshev_dos(cheb, n, d, t, g["delta_degrees"])[1], g["delta_density"])
    # Delta-Gauss-Legendre (dgl.py:42-132)
    np.testing.assert_array_equal(O.dgl_dos(leg, n, d, float(g["dgl_sigma"]), t)[1], g["dgl_density"])
    for i in range(4):
        ga, ps, ef = O.dgl_gamma_table(np.array([float(g[f"dglcoef{i}_t"])]), 0.05, degree)
        k = int(ef[0])
        assert k == int(g[f"dglcoef{i}_effective"])
        np.testing.assert_array_equal(ga[: k + 1, 0], g[f"dglcoef{i}_gamma"])
        np.testing.assert_array_equal(ps[: k + 1, 0], g[f"dglcoef{i}_psi"])


def _interval_matrices(g):
    import scipy.sparse as sp

    return {"c1": W.build_matrix("C1").csr, "c2": W.build_matrix("C2").csr, "dense20": sp.csr_array(g["dense20"]),
            "diag10": sp.csr_array(np.diag(np.arange(1.0, 11.0))), "diag3": sp.csr_array(np.diag([-3.0, 0.0, 5.0]))}


def test_oracle_interval_matches_reference(golden):
    """estimate_spectral_interval / ritz_residual_bounds (matrix.py:207-241, lanczos.py:162-167)."""
    g = golden("interval")
    mats = _interval_matrices(g)
    for i in range(int(g["runs"])):
        csr = mats[str(g[f"run{i}_matrix"])]
        steps, margin = int(g[f"run{i}_steps"]), float(g[f"run{i}_margin"])
        lb, ub = O.estimate_spectral_interval(csr, steps, margin)
        assert (lb, ub) == (float(g[f"run{i}_lb"]), float(g[f"run{i}_ub"]))
        v0 = O.draw_probe("gaussian", 0, csr.shape[0], 0, stream=0xB0)
        a, b, bn, _, _ = O.lanczos_factorize(csr, v0, min(steps, csr.shape[0]))
        theta, resid = O.ritz_residual_bounds(a, b, bn)
        np.testing.assert_array_equal(theta, g[f"run{i}_theta"])
        np.testing.assert_array_equal(resid, g[f"run{i}_resid"])


HAYDOCK_CASES = {"haydock_small": lambda: W.anderson_3d(8), "haydock_c4": lambda: W.build_matrix("C4")}


@pytest.mark.parametrize("name", list(HAYDOCK_CASES))
def test_oracle_haydock_matches_reference(golden, name):
    """haydock_dos + resolvent routes (lanczos.py:222-293)."""
    g = golden(name)
    if name == "haydock_c4":
        # the full run takes ~1 min of CPU: check the resolvent routes only
        np.testing.assert_array_equal(O.continued_fraction_resolvent(g["alpha0"], g["beta0"], g["z"]), g["cf"])
        w0, wl = O.tridiagonal_resolvent_first(g["alpha0"], g["beta0"], g["z"])
        np.testing.assert_array_equal(w0, g["w_first"])
        np.testing.assert_array_equal(wl, g["w_last"])
        return
    op = HAYDOCK_CASES[name]()
    assert csr_digest(op.csr) == str(g["matrix_sha256"])
    dens, trunc = O.haydock_dos(op.csr, int(g["steps"]), str(g["kind"]), 0, int(g["n_vec"]), float(g["eta"]),
                                g["grid"])
    np.testing.assert_array_equal(dens, g["density"])
    assert trunc == float(g["trunc"])
    np.testing.assert_array_equal(O.continued_fraction_resolvent(g["alpha0"], g["beta0"], g["z"]), g["cf"])
    w0, wl = O.tridiagonal_resolvent_first(g["alpha0"], g["beta0"], g["z"])
    np.testing.assert_array_equal(w0, g["w_first"])
    np.testing.assert_array_equal(wl, g["w_last"])

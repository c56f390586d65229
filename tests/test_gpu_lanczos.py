"""Lanczos quadrature on the GPU: reference contract (pkg/tests/test_lanczos.py
:43-204, test_acceptance.py:157-196) + parity with golden outputs and the oracle."""

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from oracle import specdens_oracle as O
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.gpu

DOS_ATOL = 1e-9


def random_symmetric(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    a = 0.5 * (a + a.T) * scale
    return sdb.SparseSymmetricMatrix.from_dense(a), a


def gaussian_kernel(x, s):
    return np.exp(-0.5 * (x / s) ** 2) / np.sqrt(2.0 * np.pi * s * s)


def test_full_run_recovers_spectrum():
    op = sdb.SparseSymmetricMatrix.from_dense(np.diag([1.0, 2.0, 3.0]))
    fact = sdb.lanczos_factorize(op, np.ones(3) / np.sqrt(3.0), 3)
    quad = sdb.ritz_quadrature(fact)
    np.testing.assert_allclose(quad.theta, [1.0, 2.0, 3.0], atol=1e-12)
    assert quad.tau_sq.sum() == pytest.approx(1.0, abs=1e-13)


def test_eigenvector_start_breaks_down():
    op = sdb.SparseSymmetricMatrix.from_dense(np.diag([1.0, 2.0, 3.0]))
    fact = sdb.lanczos_factorize(op, np.array([0.0, 1.0, 0.0]), 3)
    assert fact.breakdown
    np.testing.assert_array_equal(fact.alpha, [2.0])
    assert fact.beta.size == 0 and fact.beta_next == 0.0


def test_full_steps_match_dense_eigenvalues():
    op, a = random_symmetric(30, 7)
    fact = sdb.lanczos_factorize(op, np.random.default_rng(11).standard_normal(30), 30)
    np.testing.assert_allclose(sdb.ritz_quadrature(fact).theta, np.linalg.eigvalsh(a), atol=1e-8)


@pytest.mark.parametrize("reorth", ["full", "selective"])
def test_factorization_identity_and_orthonormality(reorth):
    op, a = random_symmetric(20, 3)
    m = 12
    fact = sdb.lanczos_factorize(op, np.random.default_rng(5).standard_normal(20), m, reorth=reorth)
    v = fact.basis
    t = np.diag(fact.alpha) + np.diag(fact.beta, 1) + np.diag(fact.beta, -1)
    resid = a @ v - v @ t
    assert np.linalg.norm(resid[:, :-1]) <= 1e-8 * np.linalg.norm(a)
    assert np.linalg.norm(resid[:, -1]) == pytest.approx(fact.beta_next, rel=1e-10)
    if reorth == "full":
        assert np.max(np.abs(v.T @ v - np.eye(m))) <= 1e-12


def test_prefix_matches_shorter_run():
    op, _ = random_symmetric(18, 9)
    v0 = np.random.default_rng(2).standard_normal(18)
    long = sdb.lanczos_factorize(op, v0, 12)
    short = sdb.lanczos_factorize(op, v0, 5)
    pre = sdb.prefix_factorization(long, 5)
    np.testing.assert_array_equal(pre.alpha, short.alpha)
    np.testing.assert_array_equal(pre.beta, short.beta)
    assert pre.beta_next == short.beta_next
    assert sdb.prefix_factorization(long, 12) is long


def test_invalid_arguments():
    op, _ = random_symmetric(6, 0)
    v0 = np.ones(6)
    for args in ((v0, 0), (v0, 7), (np.zeros(6), 3)):
        with pytest.raises(ValueError):
            sdb.lanczos_factorize(op, *args)
    with pytest.raises(ValueError):
        sdb.lanczos_factorize(op, v0, 3, reorth="lazy")


def test_ritz_small_cases():
    op = sdb.SparseSymmetricMatrix.from_dense(np.array([[5.0]]))
    quad = sdb.ritz_quadrature(sdb.lanczos_factorize(op, np.array([2.0]), 1))
    np.testing.assert_array_equal(quad.theta, [5.0])
    np.testing.assert_array_equal(quad.tau_sq, [1.0])
    two = sdb.TridiagonalFactorization(alpha=np.zeros(2), beta=np.ones(1), beta_next=0.0)
    quad = sdb.ritz_quadrature(two)
    np.testing.assert_allclose(quad.theta, [-1.0, 1.0], atol=1e-15)
    np.testing.assert_allclose(quad.tau_sq, [0.5, 0.5], atol=1e-15)


def test_quadrature_is_exact_to_degree_2m_minus_1():
    for seed in (21, 22, 23):
        op, a = random_symmetric(20, seed)
        rng = np.random.default_rng(4)
        v0 = rng.standard_normal(20)
        v0 /= np.linalg.norm(v0)
        quad = sdb.ritz_quadrature(sdb.lanczos_factorize(op, v0, 5))
        w = v0.copy()
        for q in range(10):
            exact = float(v0 @ w)
            approx = float(np.sum(quad.tau_sq * quad.theta**q))
            assert abs(approx - exact) <= 1e-9 * max(abs(exact), 1.0)
            w = a @ w


def test_ritz_weights_sum_to_one_and_match_lapack():
    rng = np.random.default_rng(123)
    for dim in range(2, 13):
        a = rng.standard_normal((dim, dim))
        op = sdb.SparseSymmetricMatrix.from_dense(0.5 * (a + a.T))
        fact = sdb.lanczos_factorize(op, rng.standard_normal(dim), dim)
        quad = sdb.ritz_quadrature(fact)
        assert abs(quad.tau_sq.sum() - 1.0) <= 1e-12
        th, tw = O.ritz_quadrature(fact.alpha, fact.beta)
        np.testing.assert_allclose(quad.theta, th, atol=1e-12)


def test_breakdown_truncation_weights():
    op = sdb.SparseSymmetricMatrix.from_dense(np.eye(3))
    fact = sdb.lanczos_factorize(op, np.array([1.0, 2.0, -1.0]), 3)
    assert fact.breakdown
    quad = sdb.ritz_quadrature(fact)
    np.testing.assert_allclose(quad.theta, [1.0], atol=1e-14)
    assert quad.tau_sq.sum() == pytest.approx(1.0, abs=1e-14)


def test_single_eigenvalue_blur_is_gaussian():
    op = sdb.SparseSymmetricMatrix.from_dense(np.array([[0.3]]))
    iv = sdb.SpectralInterval(-1.0, 1.0)
    grid = sdb.interval_grid(iv, 201)
    est = sdb.lanczos_dos(op, iv, 1, sdb.ProbeVectorSource("gaussian", seed=0, dim=1), 2, sigma=0.2, grid=grid)
    np.testing.assert_allclose(est.density, gaussian_kernel(grid - 0.3, 0.2), rtol=1e-13)


@pytest.mark.parametrize("n", [24, 200])
def test_exhaustive_full_depth_reproduces_blurred_spectrum(n):
    op, a = random_symmetric(n, 17 if n == 24 else 0)
    lam = np.linalg.eigvalsh(a)
    iv = sdb.SpectralInterval(lam[0] - 0.5, lam[-1] + 0.5)
    grid = sdb.interval_grid(iv, 300 if n == 24 else 500)
    s = 0.1
    est = sdb.lanczos_dos(op, iv, n, sdb.ProbeVectorSource("basis", seed=0, dim=n), n, sigma=s, grid=grid)
    oracle = gaussian_kernel(grid[:, None] - lam[None, :], s).mean(axis=1)
    assert np.max(np.abs(est.density - oracle)) <= (1e-10 if n == 24 else 1e-9)


def test_pool_and_blur_match_oracle():
    rng = np.random.default_rng(3)
    quads = [sdb.RitzQuadrature(theta=np.sort(rng.standard_normal(k)), tau_sq=rng.random(k)) for k in (5, 9, 1, 7)]
    pooled = sdb.pool_ritz_quadratures(quads)
    th, tw = O.pool([(q.theta, q.tau_sq) for q in quads])
    np.testing.assert_array_equal(pooled.theta, th)
    np.testing.assert_allclose(pooled.tau_sq, tw, rtol=1e-15)
    grid = np.linspace(-3, 3, 301)
    dens = sdb.blur_nodes(pooled.theta, pooled.tau_sq, grid, sdb.RegularizationKernel("gaussian", 0.2))
    np.testing.assert_allclose(dens, O.blur_nodes(th, tw, grid, 0.2), rtol=0, atol=1e-14)


def _lanczos_golden(golden, name, op):
    g = golden(name)
    iv = sdb.SpectralInterval(float(g["lb"]), float(g["ub"]))
    src = sdb.ProbeVectorSource(str(g["kind"]), seed=0, dim=op.dim)
    est = sdb.lanczos_dos(op, iv, int(g["steps"]), src, int(g["n_vec"]), float(g["sigma"]), g["grid"])
    assert np.max(np.abs(est.density - g["density"])) <= DOS_ATOL
    np.testing.assert_allclose(est.params["ritz_nodes"], g["ritz_nodes"], rtol=0, atol=1e-10)
    est2 = sdb.estimate_dos(op, iv, "lanczos", int(g["steps"]), src, int(g["n_vec"]), sigma=float(g["sigma"]),
                            grid_points=int(g["n_pts"]))
    assert np.max(np.abs(est2.density - g["estimate_density"])) <= DOS_ATOL
    assert est2.params["matvec_count"] == int(g["estimate_matvec_count"])
    for l in range(g["alpha"].shape[0]):
        f = sdb.lanczos_factorize(op, src.draw(l), int(g["steps"]))
        scale = np.max(np.abs(g["alpha"][l]))
        assert np.max(np.abs(f.alpha - g["alpha"][l])) <= 1e-10 * scale
        assert np.max(np.abs(f.beta - g["beta"][l])) <= 1e-10 * scale


def test_golden_lanczos_small(golden):
    _lanczos_golden(golden, "lanczos_small", W.anderson_3d(8))


def test_golden_c4_subset(golden):
    op = W.build_matrix("C4")
    _lanczos_golden(golden, "c4_subset", op)
    _lanczos_golden(golden, "c4_subset", sdb.SparseSymmetricMatrix(csr=op.csr))


def test_lanczos_nonfinite_raises():
    op = sdb.SparseSymmetricMatrix.from_dense(np.array([[np.inf, 0.0], [0.0, 1.0]]))
    with pytest.raises(sdb.NumericalFailure, match="non-finite Lanczos"):
        sdb.lanczos_factorize(op, np.ones(2), 2)


@pytest.mark.parametrize("steps", [5, 40, 100, 300])
def test_fused_cgs2_pass_matches_four_pass_schedule(monkeypatch, steps):
    """The fused update+projection pass (K5c) against the unfused 4-pass CGS2
    schedule on the same probes: same math, only the summation order differs.
    300 steps exceeds the fused kernel's register range and takes the fallback."""
    op = W.anderson_3d(12)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("gaussian", seed=3, dim=op.dim)
    grid = sdb.interval_grid(iv, 256)
    monkeypatch.setenv("SDB_LZ_FUSED", "1")
    fused = sdb.lanczos_dos(op, iv, steps, src, 70, 0.05, grid)
    monkeypatch.setenv("SDB_LZ_FUSED", "0")
    plain = sdb.lanczos_dos(op, iv, steps, src, 70, 0.05, grid)
    assert np.max(np.abs(fused.density - plain.density)) <= 1e-10
    np.testing.assert_allclose(fused.params["ritz_nodes"], plain.params["ritz_nodes"], rtol=0, atol=1e-10)
    if steps <= 100:
        monkeypatch.setenv("SDB_LZ_FUSED", "1")
        for l in (0, 69):
            alpha, beta = O.lanczos_factorize(op.csr, src.draw(l), steps)[:2]
            f = sdb.lanczos_factorize(op, src.draw(l), steps)
            scale = np.max(np.abs(alpha))
            assert np.max(np.abs(f.alpha - alpha)) <= 1e-10 * scale
            assert np.max(np.abs(f.beta - beta)) <= 1e-10 * scale


@pytest.mark.parametrize("steps", [5, 40, 100, 300])
def test_gram_two_pass_reorthogonalisation_matches_three_pass(monkeypatch, steps):
    """The two-pass full reorthogonalisation (projection + Gram column, h = 2 h1 - G h1,
    one update; default for n >= 16384 and steps <= n / 64) against the three-pass CGS2
    schedule and the oracle on the same probes; 300 steps is past the fused three-pass
    kernel's range (the comparison run finishes on the 4-pass fallback)."""
    op = W.anderson_3d(12)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("gaussian", seed=3, dim=op.dim)
    grid = sdb.interval_grid(iv, 256)
    monkeypatch.setenv("SDB_LZ_GRAM", "1")
    gram = sdb.lanczos_dos(op, iv, steps, src, 70, 0.05, grid)
    monkeypatch.setenv("SDB_LZ_GRAM", "0")
    plain = sdb.lanczos_dos(op, iv, steps, src, 70, 0.05, grid)
    assert np.max(np.abs(gram.density - plain.density)) <= 1e-10
    np.testing.assert_allclose(gram.params["ritz_nodes"], plain.params["ritz_nodes"], rtol=0, atol=1e-10)
    monkeypatch.setenv("SDB_LZ_GRAM", "1")
    if steps <= 100:
        for l in (0, 69):
            alpha, beta = O.lanczos_factorize(op.csr, src.draw(l), steps)[:2]
            f = sdb.lanczos_factorize(op, src.draw(l), steps)
            scale = np.max(np.abs(alpha))
            assert np.max(np.abs(f.alpha - alpha)) <= 1e-10 * scale
            assert np.max(np.abs(f.beta - beta)) <= 1e-10 * scale
            v = f.basis
            assert np.max(np.abs(v.T @ v - np.eye(v.shape[1]))) <= 1e-12
    # a shorter run is an exact prefix of a longer one under the same schedule
    v0 = src.draw(1)
    long = sdb.lanczos_factorize(op, v0, min(steps, 60))
    short = sdb.lanczos_factorize(op, v0, min(steps, 60) // 2 + 1)
    np.testing.assert_array_equal(long.alpha[:short.alpha.size], short.alpha)


def test_gram_two_pass_breakdown_and_frozen_probes(monkeypatch):
    """Invariant-subspace breakdown under the two-pass schedule: a matrix with three
    distinct eigenvalues stops after three steps (beta <= 1e-13 scale), like the
    reference; an eigenvector start stops after one."""
    monkeypatch.setenv("SDB_LZ_GRAM", "1")
    n = 4000
    rng = np.random.default_rng(1)
    d = rng.choice([-0.7, 0.1, 0.6], size=n)
    import scipy.sparse as sp
    op = sdb.SparseSymmetricMatrix(csr=sp.diags(d).tocsr())
    f = sdb.lanczos_factorize(op, rng.standard_normal(n), 8)
    assert f.breakdown and f.alpha.size == 3
    np.testing.assert_allclose(np.sort(sdb.ritz_quadrature(f).theta), [-0.7, 0.1, 0.6], atol=1e-12)
    e = np.zeros(n)
    e[5] = 1.0
    f1 = sdb.lanczos_factorize(op, e, 4)
    assert f1.breakdown and f1.alpha.size == 1

"""Spectral-interval estimation on the GPU: the 20-step Lanczos
run, Ritz values and residual bounds on the device (estimate_spectral_interval,
matrix.py:207-241; ritz_residual_bounds, lanczos.py:162-167).

Reference contract tests restated from pkg/tests/test_matrix.py:176-214; parity
against the reference's outputs (tests/golden/interval.npz).  The GPU Lanczos
basis differs from the reference's BLAS-ordered one in the last bits, so the
bounds are compared to 1e-9 of the spectral scale.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_interval_diag_full_steps_contains_spectrum():
    mat = sdb.SparseSymmetricMatrix.from_dense(np.diag(np.arange(1.0, 11.0)))
    iv = sdb.estimate_spectral_interval(mat, lanczos_steps=10, seed=0)
    assert iv.lambda_lb <= 1.0 and iv.lambda_ub >= 10.0


def test_interval_three_steps_brackets_extremes():
    mat = sdb.SparseSymmetricMatrix.from_dense(np.diag([-3.0, 0.0, 5.0]))
    iv = sdb.estimate_spectral_interval(mat, lanczos_steps=3, seed=0)
    assert iv.lambda_lb <= -3.0 and iv.lambda_ub >= 5.0


def test_interval_full_steps_tight_without_margin():
    rng = np.random.default_rng(11)
    a = rng.standard_normal((20, 20))
    mat = sdb.SparseSymmetricMatrix.from_dense(a + a.T)
    ev = np.linalg.eigvalsh(a + a.T)
    iv = sdb.estimate_spectral_interval(mat, lanczos_steps=20, margin=0.0, seed=0)
    scale = max(abs(ev[0]), abs(ev[-1]))
    assert abs(iv.lambda_lb - ev[0]) <= 1e-8 * scale
    assert abs(iv.lambda_ub - ev[-1]) <= 1e-8 * scale


def test_interval_contains_laplacian_spectrum():
    mat = W.generate_modified_laplacian_2d(10, 5)
    ev = np.linalg.eigvalsh(mat.csr.toarray())
    iv = sdb.estimate_spectral_interval(mat)
    assert iv.lambda_lb <= ev[0] and iv.lambda_ub >= ev[-1]


def test_interval_errors():
    mat = sdb.SparseSymmetricMatrix.from_dense(np.eye(4))
    with pytest.raises(ValueError):
        sdb.estimate_spectral_interval(mat, lanczos_steps=1)
    bad = sdb.SparseSymmetricMatrix.from_dense(np.array([[np.inf, 0.0], [0.0, 1.0]]))
    with pytest.raises(sdb.NumericalFailure):
        sdb.estimate_spectral_interval(bad)


def test_residual_bounds_single_step():
    f = sdb.TridiagonalFactorization(alpha=np.array([2.5]), beta=np.zeros(0), beta_next=-0.75)
    theta, resid = sdb.ritz_residual_bounds(f)
    np.testing.assert_array_equal(theta, [2.5])
    np.testing.assert_array_equal(resid, [0.75])


def test_interval_matches_reference(golden):
    g = golden("interval")
    mats = {"c1": W.build_matrix("C1"), "c2": W.build_matrix("C2"),
            "dense20": sdb.SparseSymmetricMatrix(csr=sp.csr_array(g["dense20"])),
            "diag10": sdb.SparseSymmetricMatrix.from_dense(np.diag(np.arange(1.0, 11.0))),
            "diag3": sdb.SparseSymmetricMatrix.from_dense(np.diag([-3.0, 0.0, 5.0]))}
    for i in range(int(g["runs"])):
        key = str(g[f"run{i}_matrix"])
        steps, margin = int(g[f"run{i}_steps"]), float(g[f"run{i}_margin"])
        iv = sdb.estimate_spectral_interval(mats[key], lanczos_steps=steps, margin=margin, seed=0)
        lb, ub = float(g[f"run{i}_lb"]), float(g[f"run{i}_ub"])
        scale = max(abs(lb), abs(ub), 1.0)
        assert abs(iv.lambda_lb - lb) <= 1e-9 * scale, (key, steps)
        assert abs(iv.lambda_ub - ub) <= 1e-9 * scale, (key, steps)
        # the Ritz values / residual bounds of the reference's own factorization
        theta_ref = g[f"run{i}_theta"]
        src = sdb.ProbeVectorSource("gaussian", seed=0, dim=mats[key].dim, stream=0xB0)
        fact = sdb.lanczos_factorize(mats[key], src.draw(0), min(steps, mats[key].dim))
        theta, resid = sdb.ritz_residual_bounds(fact)
        assert np.max(np.abs(theta - theta_ref)) <= 1e-9 * scale
        assert np.max(np.abs(resid - g[f"run{i}_resid"])) <= 1e-7 * scale

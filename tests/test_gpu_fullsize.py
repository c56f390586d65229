"""BASELINE.json's full sizes on the GPU, checked against the C oracle on probe
subsets (draw(l) is independent of the other probes, stochastic.py:22-27, and
moments are exact prefixes, kpm.py:49-59) plus size-independent properties:

* C2 bench workload exactly (Anderson 64^3 CSR, 64 Rademacher probes, M = 500
  doubling, Jackson, 2000 points) end to end through estimate_dos against the
  C oracle's moments of all 64 probes and the NumPy oracle's DOS of those.
* C3 (n = 1e6, ~61M nnz CSR, KPM M = 1000, 128 Gaussian probes, band + far
  kernel): per-probe moments of probes {0, 1} at the FULL M = 1000 against the
  C oracle; zeta_0 = host mean |v|^2, |zeta_k| <= zeta_0; the DOS stage fed
  with the GPU moments against the oracle's evaluation of the same moments.
* C5 (256^3 27-point stencil, M = 2000, 32 Rademacher probes): probes {0, 1}
  at M = 200 against the C oracle's stencil path (pinned to its CSR path,
  tests/test_oracle_stencil.py); zeta_0 = n exactly, |zeta_k| <= n, direct ==
  doubling on a prefix, row-partitioned run == whole-grid run.
Tolerances (north star): moments max|dz|/max|z| <= 1e-10, DOS max-abs <= 1e-9.
"""

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from oracle import specdens_oracle as O
from paper_1308_5467_b200 import _native
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.rowpart import rowpartition_moments

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b))


@pytest.fixture(scope="module")
def c3():
    mat = W.build_matrix("C3")
    return mat, W.gershgorin_interval(mat)


def test_c3_full_config_properties_and_oracle_prefix(c3):
    from oracle import c_oracle

    mat, iv = c3
    cfg = W.CONFIGS["C3"]
    src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=mat.dim)
    run = E.run_chebyshev(sdb.apply_spectral_map(mat, iv), cfg.degree, src, cfg.n_vec, _native.SDB_CHEB_DOUBLING)
    zpp = run.zeta_pp.cpu().numpy()
    assert zpp.shape == (cfg.n_vec, cfg.degree + 1) and np.all(np.isfinite(zpp))
    norms = np.array([np.dot(v, v) for v in (src.draw(l) for l in range(cfg.n_vec))])
    assert rel(zpp[:, 0], norms) <= 1e-12
    assert np.all(np.abs(zpp) <= zpp[:, :1] * (1 + 1e-10))  # |T_k| <= 1 on the mapped spectrum
    assert c_oracle.available()
    probes = np.array([src.draw(l) for l in (0, 1)])
    ref = c_oracle.cheb_moments(mat.csr, iv.center, iv.halfwidth, cfg.degree, probes, mode="doubling", threads=2)
    for l in (0, 1):
        assert rel(zpp[l], ref[l]) <= 1e-10
    est = sdb.estimate_dos(mat, iv, "kpm-jackson", cfg.degree, src, cfg.n_vec, grid_points=cfg.grid_points,
                           product_formula=True)
    zeta = est.params["moments"]
    assert rel(zeta, zpp.mean(axis=0)) <= 1e-13
    coeffs = O.moments_to_coefficients(zeta, mat.dim, "jackson")
    _, dens = O.evaluate_kpm_dos(coeffs, iv.halfwidth, O.unit_grid(cfg.grid_points))
    assert np.max(np.abs(est.density - dens)) <= 1e-9


def test_c5_full_config_properties_and_row_partition():
    op = W.build_matrix("C5")
    iv = W.gershgorin_interval(op)
    cfg = W.CONFIGS["C5"]
    src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=op.dim)
    mapped = sdb.apply_spectral_map(op, iv)
    run = E.run_chebyshev(mapped, cfg.degree, src, cfg.n_vec, _native.SDB_CHEB_DOUBLING)
    zpp = run.zeta_pp.cpu().numpy()
    n = float(op.dim)
    from oracle import c_oracle

    assert c_oracle.available()
    probes = np.array([src.draw(l) for l in (0, 1)])
    ref = c_oracle.stencil_moments(op, iv.center, iv.halfwidth, 200, probes, mode="doubling", threads=2)
    for l in (0, 1):
        assert rel(zpp[l, :201], ref[l]) <= 1e-10
    assert np.all(np.isfinite(zpp))
    assert np.all(zpp[:, 0] == n)  # Rademacher probes: v.v = n exactly
    assert np.all(np.abs(zpp) <= n * (1 + 1e-10))
    direct = E.run_chebyshev(mapped, 40, src, cfg.n_vec, _native.SDB_CHEB_DIRECT).zeta_pp.cpu().numpy()
    assert rel(zpp[:, :41], direct) <= 1e-10
    part = rowpartition_moments(op, iv, 200, src, cfg.n_vec, n_slabs=2, exchange="copy",
                                layout="planes").cpu().numpy()
    assert rel(part, zpp[:, :201]) <= 1e-12


def test_c4_full_config_quadrature_properties():
    """C4 (Lanczos m = 100 with full reorthogonalisation on the C2 matrix, 128
    Gaussian probes, sigma = 0.01, 2000 points): pooled Gauss weights sum to 1
    (each probe's tau^2 sums to |e_1|^2 = 1), nodes are sorted and inside the
    Gershgorin interval, the density is the oracle's blur of the GPU's nodes, and
    probe 0's tridiagonal matches the oracle (the golden c4_subset pins 4 probes)."""
    op = W.build_matrix("C4")
    iv = W.gershgorin_interval(op)
    cfg = W.CONFIGS["C4"]
    src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=op.dim)
    grid = sdb.interval_grid(iv, cfg.grid_points)
    est = sdb.lanczos_dos(op, iv, cfg.degree, src, cfg.n_vec, cfg.sigma, grid)
    nodes, weights = est.params["ritz_nodes"], est.params["ritz_weights"]
    assert len(nodes) == cfg.degree * cfg.n_vec
    assert abs(np.sum(weights) - 1.0) <= 1e-12
    assert np.all(np.diff(nodes) >= 0)
    assert nodes[0] >= iv.lambda_lb - 1e-9 and nodes[-1] <= iv.lambda_ub + 1e-9
    assert np.max(np.abs(est.density - O.blur_nodes(nodes, weights, grid, cfg.sigma))) <= 1e-9
    alpha, beta = O.lanczos_factorize(op.csr, src.draw(0), cfg.degree)[:2]
    f = sdb.lanczos_factorize(op, src.draw(0), cfg.degree)
    assert rel(f.alpha, alpha) <= 1e-10 and np.max(np.abs(f.beta - beta)) <= 1e-10 * np.max(np.abs(alpha))


def test_c2_bench_workload_end_to_end():
    """bench.py --config C2 exactly: CSR input (detected stencil), 64 Rademacher
    probes, M = 500 product formula, Jackson, 2000 points."""
    from oracle import c_oracle

    op = W.build_matrix("C2")
    mat = sdb.SparseSymmetricMatrix(csr=op.csr)
    iv = W.gershgorin_interval(mat)
    cfg = W.CONFIGS["C2"]
    src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=mat.dim)
    est = sdb.estimate_dos(mat, iv, "kpm-jackson", cfg.degree, src, cfg.n_vec, grid_points=cfg.grid_points,
                           product_formula=True)
    probes = np.array([src.draw(l) for l in range(cfg.n_vec)])
    ref = c_oracle.cheb_moments(mat.csr, iv.center, iv.halfwidth, cfg.degree, probes, mode="doubling")
    zeta = ref.mean(axis=0)
    assert rel(est.params["moments"], zeta) <= 1e-10
    _, dens = O.evaluate_kpm_dos(O.moments_to_coefficients(zeta, mat.dim, "jackson"), iv.halfwidth,
                                 O.unit_grid(cfg.grid_points))
    assert np.max(np.abs(est.density - dens)) <= 1e-9

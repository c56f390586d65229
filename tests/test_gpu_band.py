"""Probe-sliced band + far kernel (band.cu, BASELINE config 3's matrix class).

* The split is made at upload only for CSR matrices with a dense, bit-exactly
  symmetric band and sorted rows; otherwise the plain CSR kernel runs.
* A row's sum runs far entries (column order) then the band, the CSR kernel in
  pure column order: w agrees to rounding, the moments with the CSR kernel's
  to 1e-13 and with the C oracle (csr_matvec order, kpm.py:96-107 / :174-189)
  within the north-star 1e-10 (max|dz|/max|z|).
* Edge cases: n not a multiple of the 128-row tile, probe counts that are not a
  multiple of the 16-column slice (1, 20, 130), every moment mode, a narrow
  band (half-width 8) on a matrix of a few tiles.
"""

import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1308_5467_b200 as sdb
from oracle import c_oracle
from paper_1308_5467_b200 import _native
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.operators import device_matrix, resolve

pytestmark = pytest.mark.gpu

MODES = {"doubling": _native.SDB_CHEB_DOUBLING, "direct": _native.SDB_CHEB_DIRECT, "legendre": _native.SDB_LEGENDRE}


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b))


def kernel_of(mat, n_vec, mode):
    import torch

    dm = device_matrix(mat, 0, E.stream_ptr(0))
    return dm, _native.load().sdb_cheb_kernel(dm.handle, n_vec, mode).decode()


def moments(mat, iv, degree, src, n_vec, mode, band=True):
    old = os.environ.get("SDB_BAND")
    os.environ["SDB_BAND"] = "1" if band else "0"
    try:
        run = E.run_chebyshev(sdb.apply_spectral_map(mat, iv), degree, src, n_vec, mode)
        return run.zeta_pp.cpu().numpy()
    finally:
        if old is None:
            os.environ.pop("SDB_BAND", None)
        else:
            os.environ["SDB_BAND"] = old


@pytest.fixture(scope="module")
def c3_small():
    mat = W.dft_like(20_011)  # not a multiple of the 128-row tile
    return mat, W.gershgorin_interval(mat)


def test_split_detected_for_c3_class(c3_small):
    mat, _ = c3_small
    dm, name = kernel_of(mat, 128, _native.SDB_CHEB_DOUBLING)
    assert dm.band_half_width == 20
    n = mat.dim
    far = mat.csr.nnz - (41 * n - 2 * sum(range(1, 21)))
    assert dm.band_far_entries == far
    assert name == "cheb_step_band"


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("n_vec", [1, 20, 128, 130])
def test_band_kernel_matches_csr_kernel(c3_small, mode, n_vec):
    mat, iv = c3_small
    src = sdb.ProbeVectorSource("gaussian", seed=3, dim=mat.dim)
    deg = 60
    a = moments(mat, iv, deg, src, n_vec, MODES[mode], band=True)
    b = moments(mat, iv, deg, src, n_vec, MODES[mode], band=False)
    assert a.shape == b.shape == (n_vec, deg + 1)
    assert rel(a, b) <= 1e-13


@pytest.mark.parametrize("mode", ["doubling", "direct"])
def test_band_kernel_matches_c_oracle(c3_small, mode):
    mat, iv = c3_small
    src = sdb.ProbeVectorSource("gaussian", seed=0, dim=mat.dim)
    deg = 300
    z = moments(mat, iv, deg, src, 32, MODES[mode])
    probes = np.array([src.draw(l) for l in range(4)])
    ref = c_oracle.cheb_moments(mat.csr, iv.center, iv.halfwidth, deg, probes, mode=mode, threads=4)
    for l in range(4):
        assert rel(z[l], ref[l]) <= 1e-10


def test_band_estimate_dos_front_door(c3_small):
    mat, iv = c3_small
    src = sdb.ProbeVectorSource("gaussian", seed=0, dim=mat.dim)
    est = sdb.estimate_dos(mat, iv, "kpm-jackson", 100, src, 16, grid_points=500, product_formula=True)
    from oracle import specdens_oracle as O

    probes = np.array([src.draw(l) for l in range(16)])
    ref = c_oracle.cheb_moments(mat.csr, iv.center, iv.halfwidth, 100, probes, mode="doubling", threads=8)
    zeta = ref.mean(axis=0)
    assert rel(est.params["moments"], zeta) <= 1e-10
    _, dens = O.evaluate_kpm_dos(O.moments_to_coefficients(zeta, mat.dim, "jackson"), iv.halfwidth,
                                 O.unit_grid(500))
    assert np.max(np.abs(est.density - dens)) <= 1e-9


def _csr(a):
    a = sp.csr_array(a)
    a.sort_indices()
    return sdb.SparseSymmetricMatrix(csr=a)


def test_no_split_when_values_not_symmetric(c3_small):
    mat, _ = c3_small
    csr = mat.csr.copy()
    row = 5000
    k = np.searchsorted(csr.indices[csr.indptr[row]:csr.indptr[row + 1]], row - 3) + csr.indptr[row]
    assert csr.indices[k] == row - 3
    csr.data = csr.data.copy()
    csr.data[k] = np.nextafter(csr.data[k], np.inf)  # one ulp off its mirror
    dm, name = kernel_of(sdb.SparseSymmetricMatrix(csr=csr), 64, _native.SDB_CHEB_DOUBLING)
    assert dm.band_half_width == 0 and name == "cheb_step_csr"


def test_no_split_without_dense_band():
    mat = W.build_matrix("C1")  # 2-D Laplacian: offsets 1 and 100 only
    dm, name = kernel_of(mat, 20, _native.SDB_CHEB_DOUBLING)
    assert dm.band_half_width == 0


def test_band_kernel_small_band_and_tail_tile():
    # 13-diagonal band plus random pairs, n = 600 (2 full 256-row tiles + an 88-row tail)
    n = 600
    rng = np.random.default_rng(7)
    dense = np.zeros((n, n))
    for d in range(0, 7):
        v = rng.standard_normal(n - d)
        dense[np.arange(n - d), np.arange(d, n)] = v
        dense[np.arange(d, n), np.arange(n - d)] = v
    for _ in range(800):
        i, j = rng.integers(0, n, 2)
        if abs(i - j) > 8:
            v = rng.standard_normal()
            dense[i, j] = dense[j, i] = v
    mat = _csr(dense)
    iv = W.gershgorin_interval(mat)
    dm, name = kernel_of(mat, 16, _native.SDB_CHEB_DOUBLING)
    assert dm.band_half_width == 8 and name == "cheb_step_band"
    src = sdb.ProbeVectorSource("rademacher", seed=1, dim=n)
    for mode in ("doubling", "direct"):
        z = moments(mat, iv, 50, src, 16, MODES[mode])
        ref = c_oracle.cheb_moments(mat.csr, iv.center, iv.halfwidth, 50, np.array([src.draw(l) for l in range(16)]),
                                    mode=mode, threads=4)
        assert rel(z, ref) <= 1e-10


def _banded(n, half_band, n_pairs, seed, heavy_row=None):
    """Dense-band symmetric matrix plus random far pairs (optionally one row with many)."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for d in range(half_band + 1):
        v = rng.standard_normal(n - d)
        i = np.arange(n - d)
        rows += [i, i + d] if d else [i]
        cols += [i + d, i] if d else [i]
        vals += [v, v] if d else [v]
    i = rng.integers(0, n, n_pairs)
    j = rng.integers(0, n, n_pairs)
    if heavy_row is not None:
        j2 = np.setdiff1d(np.arange(n), np.arange(heavy_row - half_band - 2, heavy_row + half_band + 3))[::3]
        i = np.concatenate([i, np.full(j2.size, heavy_row)])
        j = np.concatenate([j, j2])
    keep = np.abs(i - j) > half_band + 1
    i, j = i[keep], j[keep]
    key = np.unique(np.minimum(i, j) * n + np.maximum(i, j))
    i, j = key // n, key % n
    v = rng.standard_normal(i.size)
    rows += [i, j]
    cols += [j, i]
    vals += [v, v]
    a = sp.coo_array((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n)).tocsr()
    a.sort_indices()
    return sdb.SparseSymmetricMatrix(csr=a)


@pytest.mark.parametrize("half_band,kernel_hb", [(6, 8), (13, 16), (22, 24), (30, 32)])
def test_every_band_half_width_instantiation(half_band, kernel_hb):
    """One kernel instantiation per supported half-width (the detected band is
    rounded up); 24 and 32 run the shallower gather ring."""
    n = 1500
    mat = _banded(n, half_band, 6 * n, seed=half_band)
    iv = W.gershgorin_interval(mat)
    dm, name = kernel_of(mat, 20, _native.SDB_CHEB_DOUBLING)
    assert dm.band_half_width == kernel_hb and name == "cheb_step_band"
    src = sdb.ProbeVectorSource("gaussian", seed=9, dim=n)
    probes = np.array([src.draw(l) for l in range(20)])
    for mode in ("doubling", "direct"):
        z = moments(mat, iv, 40, src, 20, MODES[mode])
        ref = c_oracle.cheb_moments(mat.csr, iv.center, iv.halfwidth, 40, probes, mode=mode, threads=4)
        assert rel(z, ref) <= 1e-10


def test_band_only_and_heavy_far_row():
    """A matrix with no far entries at all (every stream is four empty batches)
    and one whose row 700 couples to ~450 far columns (a 100+-batch chunk next
    to near-empty ones)."""
    n = 1400
    for mat in (_banded(n, 10, 0, seed=1), _banded(n, 10, 2 * n, seed=2, heavy_row=700)):
        iv = W.gershgorin_interval(mat)
        dm, name = kernel_of(mat, 16, _native.SDB_CHEB_DOUBLING)
        assert name == "cheb_step_band"
        src = sdb.ProbeVectorSource("rademacher", seed=3, dim=n)
        probes = np.array([src.draw(l) for l in range(16)])
        z = moments(mat, iv, 60, src, 16, MODES["doubling"])
        ref = c_oracle.cheb_moments(mat.csr, iv.center, iv.halfwidth, 60, probes, mode="doubling", threads=4)
        assert rel(z, ref) <= 1e-10

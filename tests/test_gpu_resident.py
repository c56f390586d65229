"""Cluster-resident recurrence for small CSR matrices (resident.cu; BASELINE config 1's class).

The whole moment run is one launch: clusters of CTAs keep their rows of w_k / w_{k-1} and their
CSR slice in shared memory and gather neighbours' rows through distributed shared memory.  Rows
accumulate in CSR storage order like the per-step CSR kernel, so both agree to rounding (1e-13);
against the oracle (kpm.py:96-107 / :174-189 / :110-124) the north-star 1e-10 holds.  Edge cases:
n below the cluster size (CTAs without rows), n not a multiple of the row block, empty rows,
probe counts that leave column pairs unused, every moment mode, degrees 1 and 2.
"""

import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1308_5467_b200 as sdb
from oracle import specdens_oracle as O
from paper_1308_5467_b200 import _native
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.operators import device_matrix

pytestmark = pytest.mark.gpu

MODES = {"doubling": _native.SDB_CHEB_DOUBLING, "direct": _native.SDB_CHEB_DIRECT, "legendre": _native.SDB_LEGENDRE}


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b))


def kernel_of(mat, n_vec, mode):
    dm = device_matrix(mat, 0, E.stream_ptr(0))
    return _native.load().sdb_cheb_kernel(dm.handle, n_vec, mode).decode()


def moments(mat, iv, degree, kind, n_vec, mode, resident=True, seed=1):
    old = os.environ.get("SDB_RESIDENT")
    os.environ["SDB_RESIDENT"] = "1" if resident else "0"
    try:
        src = sdb.ProbeVectorSource(kind, seed=seed, dim=mat.dim)
        run = E.run_chebyshev(sdb.apply_spectral_map(mat, iv), degree, src, n_vec, mode)
        return run.zeta_pp.cpu().numpy()
    finally:
        if old is None:
            os.environ.pop("SDB_RESIDENT", None)
        else:
            os.environ["SDB_RESIDENT"] = old


def irregular_symmetric(n, seed, max_per_row=12):
    """Random symmetric CSR with uneven rows (some empty off-diagonals, some without a diagonal)."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        k = int(rng.integers(0, max_per_row))
        for j in rng.integers(0, n, size=k):
            v = rng.standard_normal()
            rows += [i, int(j)]
            cols += [int(j), i]
            vals += [v, v]
    keep = rng.random(n) < 0.8
    d = rng.uniform(-2, 2, n)
    rows += list(np.nonzero(keep)[0])
    cols += list(np.nonzero(keep)[0])
    vals += list(d[keep])
    a = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    a.sum_duplicates()
    a.sort_indices()
    return sdb.SparseSymmetricMatrix(csr=a)


def test_config1_runs_resident_and_matches_the_oracle():
    mat = W.build_matrix("C1")
    iv = W.gershgorin_interval(mat)
    cfg = W.CONFIGS["C1"]
    for name, mode in MODES.items():
        assert kernel_of(mat, cfg.n_vec, mode) == "cheb_resident", name
    for name, omode in (("direct", "direct"), ("doubling", "product")):
        got = moments(mat, iv, cfg.degree, "gaussian", cfg.n_vec, MODES[name], seed=0)
        ref = O.chebyshev_moments(mat, iv.center, iv.halfwidth, cfg.degree, "gaussian", 0, cfg.n_vec, mode=omode)
        assert rel(got, ref) <= 1e-10, name


@pytest.mark.parametrize("mode", ["doubling", "direct", "legendre"])
@pytest.mark.parametrize("n,n_vec", [(3, 2), (15, 1), (17, 5), (100, 20), (1000, 64), (3001, 7), (4097, 130)])
def test_resident_matches_the_per_step_csr_kernel(mode, n, n_vec):
    mat = irregular_symmetric(n, seed=n)
    iv = W.gershgorin_interval(mat)
    m = MODES[mode]
    if n_vec <= 64:
        assert kernel_of(mat, n_vec, m) == "cheb_resident"
    elif kernel_of(mat, n_vec, m) != "cheb_resident":
        pytest.skip("block too wide for one wave of clusters")
    for degree in (1, 2, 31):
        a = moments(mat, iv, degree, "gaussian", n_vec, m, resident=True)
        b = moments(mat, iv, degree, "gaussian", n_vec, m, resident=False)
        assert a.shape == b.shape
        assert rel(a, b) <= 1e-13, (mode, n, n_vec, degree)


def test_resident_front_door_and_matvec_count():
    mat = W.build_matrix("C1")
    iv = W.gershgorin_interval(mat)
    src = sdb.ProbeVectorSource("gaussian", seed=0, dim=mat.dim)
    for pf in (False, True):
        est = sdb.estimate_dos(mat, iv, "kpm-jackson", 100, src, 20, grid_points=1000, product_formula=pf)
        per = O.chebyshev_moments(mat, iv.center, iv.halfwidth, 100, "gaussian", 0, 20,
                                  mode="product" if pf else "direct")
        zeta = O.average_moments(per)
        assert rel(est.params["moments"], zeta) <= 1e-10
        _, dens = O.evaluate_kpm_dos(O.moments_to_coefficients(zeta, mat.dim, "jackson"), iv.halfwidth,
                                     O.unit_grid(1000))
        assert np.max(np.abs(est.density - dens)) <= 1e-9
        assert est.params["matvec_count"] == (20 * 50 if pf else 20 * 100)


def test_resident_is_repeatable():
    mat = irregular_symmetric(2500, seed=9)
    iv = W.gershgorin_interval(mat)
    first = moments(mat, iv, 80, "rademacher", 20, MODES["doubling"])
    for _ in range(4):
        np.testing.assert_array_equal(moments(mat, iv, 80, "rademacher", 20, MODES["doubling"]), first)


def test_large_or_split_matrices_keep_their_kernels():
    big = W.dft_like(20_011)
    assert kernel_of(big, 16, MODES["doubling"]) == "cheb_step_band"
    op = W.anderson_3d(16)
    assert "zmarch" in kernel_of(op, 16, MODES["doubling"])

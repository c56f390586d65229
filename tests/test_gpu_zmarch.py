"""TMA z-march step kernel (zmarch.cu): parity with the oracle and with the
row-panel grid kernel, for every tile configuration, both moment modes, the
7-point star and the 27-point box, z segmentation, persistent-grid sizes and
the shallowest ring.  Tolerances as elsewhere: moments max|dz|/max|z| <= 1e-10.
"""

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from oracle import specdens_oracle as O
from paper_1308_5467_b200 import _native
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.operators import StencilOperator

pytestmark = pytest.mark.gpu

MOMENT_RTOL = 1e-10
ZMARCH = ("cheb_step_zmarch", "cheb_step2_zmarch")
FACE = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]


def make_stencil(shape, kind, seed):
    rng = np.random.default_rng(seed)
    n = shape[0] * shape[1] * shape[2]
    if kind == "face7":
        w = rng.uniform(-1.0, 1.0, 3)
        weights = [w[0], w[0], w[1], w[1], w[2], w[2]]
        return StencilOperator(shape, FACE, weights, rng.uniform(-2.0, 2.0, n))
    ref = W.stencil27_3d(4, seed=seed)  # symmetric 26-offset set with random weights
    return StencilOperator(shape, ref.offsets, ref.weights, rng.uniform(-1.0, 1.0, n) + ref.diag[0])


def kernel_name(op, n_vec, mode):
    from paper_1308_5467_b200.operators import device_matrix, resolve

    dm = device_matrix(resolve(op).base, 0, E.stream_ptr(0))
    return _native.load().sdb_cheb_kernel(dm.handle, n_vec, mode).decode()


def per_probe(op, iv, degree, src, n_vec, mode):
    run = E.run_chebyshev(sdb.apply_spectral_map(op, iv), degree, src, n_vec, mode)
    return run.zeta_pp.cpu().numpy()


def rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


# (shape, kind, n_vec, forced configuration, extra env)
CASES = [
    ((8, 8, 5), "face7", 8, 5, {}),
    ((16, 8, 7), "box27", 16, 5, {}),
    ((8, 8, 6), "box27", 20, 5, {"SDB_ZM_R": "3"}),
    ((16, 16, 6), "box27", 64, 0, {}),
    ((16, 16, 12), "face7", 64, 0, {"SDB_ZM_NZS": "3", "SDB_ZM_GRID": "16"}),
    ((32, 8, 4), "face7", 12, 1, {}),
    ((32, 8, 9), "box27", 12, 1, {"SDB_ZM_NZS": "2"}),
    ((32, 4, 9), "box27", 32, 2, {"SDB_ZM_GRID": "4"}),
    ((8, 16, 3), "face7", 48, 3, {}),
    ((8, 8, 10), "box27", 48, 3, {"SDB_ZM_NZS": "4", "SDB_ZM_R": "4"}),
    ((8, 8, 7), "face7", 16, 6, {}),
    ((16, 16, 5), "box27", 100, 4, {}),
]


@pytest.mark.parametrize("shape,kind,n_vec,cfg,env", CASES)
def test_zmarch_matches_oracle_and_grid_kernel(monkeypatch, shape, kind, n_vec, cfg, env):
    op = make_stencil(shape, kind, seed=sum(shape) + n_vec)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("gaussian", seed=1, dim=op.dim)
    degree = 17
    monkeypatch.setenv("SDB_ZM_CFG", str(cfg))
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for mode, omode in ((_native.SDB_CHEB_DOUBLING, "doubling"), (_native.SDB_CHEB_DIRECT, "direct")):
        assert kernel_name(op, n_vec, mode) in ZMARCH
        z = per_probe(op, iv, degree, src, n_vec, mode)
        ref = np.array(O.chebyshev_moments(op, iv.center, iv.halfwidth, degree, "gaussian", 1, n_vec, mode=omode))
        assert rel(z, ref) <= MOMENT_RTOL, (mode, rel(z, ref))
        monkeypatch.setenv("SDB_ZMARCH", "0")
        assert kernel_name(op, n_vec, mode) not in ZMARCH
        zg = per_probe(op, iv, degree, src, n_vec, mode)
        monkeypatch.delenv("SDB_ZMARCH")
        # same w_{k+1} bits; only the dot-product reduction trees differ
        assert rel(z, zg) <= 1e-13, (mode, rel(z, zg))


def test_zmarch_c2_full_probe_block():
    """C2 geometry (64^3 Anderson, 64 Rademacher probes) against the grid kernel
    and the oracle on two probes, degree 60."""
    import os

    op = W.build_matrix("C2")
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim)
    mode = _native.SDB_CHEB_DOUBLING
    assert kernel_name(op, 64, mode) == "cheb_step_zmarch"
    z = per_probe(op, iv, 60, src, 64, mode)
    os.environ["SDB_ZMARCH"] = "0"
    try:
        zg = per_probe(op, iv, 60, src, 64, mode)
    finally:
        del os.environ["SDB_ZMARCH"]
    assert rel(z, zg) <= 1e-13
    ref = np.array(O.chebyshev_moments(op, iv.center, iv.halfwidth, 60, "rademacher", 0, 2, mode="doubling"))
    assert rel(z[:2], ref) <= MOMENT_RTOL


def test_zmarch_estimate_dos_end_to_end():
    """The public front door on a z-march-eligible stencil matches the oracle DOS."""
    op = make_stencil((16, 16, 8), "box27", seed=3)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=2, dim=op.dim)
    est = sdb.estimate_dos(op, iv, "kpm-jackson", 40, src, 32, grid_points=300, product_formula=True)
    zeta = O.average_moments(O.chebyshev_moments(op, iv.center, iv.halfwidth, 40, "rademacher", 2, 32,
                                                 mode="doubling"))
    assert rel(est.params["moments"], zeta) <= MOMENT_RTOL
    _, dens = O.evaluate_kpm_dos(O.moments_to_coefficients(zeta, op.dim, "jackson"), iv.halfwidth, O.unit_grid(300))
    assert np.max(np.abs(est.density - dens)) <= 1e-9


# fused pairs (cheb_step2_zmarch, doubling mode, opt-in) against single z-march steps:
# same w bits, so moments agree to the reduction-order level; every step-count
# parity (degree 1..4 and odd/even tails), both shapes, every fused tile config
FUSED_CASES = [
    ((16, 16, 8), "face7", 64, 3, 17),
    ((16, 16, 8), "box27", 64, 3, 16),
    ((16, 16, 9), "box27", 32, 0, 3),
    ((32, 8, 6), "face7", 16, 2, 4),
    ((8, 8, 5), "box27", 8, 5, 2),
    ((8, 8, 4), "face7", 8, 5, 1),
    ((16, 8, 12), "box27", 16, 0, 23),
]


@pytest.mark.parametrize("shape,kind,n_vec,cfg,degree", FUSED_CASES)
def test_fused_pairs_match_single_steps(monkeypatch, shape, kind, n_vec, cfg, degree):
    op = make_stencil(shape, kind, seed=7 + n_vec)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("gaussian", seed=3, dim=op.dim)
    mode = _native.SDB_CHEB_DOUBLING
    monkeypatch.setenv("SDB_ZM_CFG", str(cfg))
    monkeypatch.setenv("SDB_ZM_FUSE", "1")
    assert kernel_name(op, n_vec, mode) == "cheb_step2_zmarch"
    z = per_probe(op, iv, degree, src, n_vec, mode)
    ref = np.array(O.chebyshev_moments(op, iv.center, iv.halfwidth, degree, "gaussian", 3, n_vec, mode="doubling"))
    assert rel(z, ref) <= MOMENT_RTOL
    monkeypatch.setenv("SDB_ZM_FUSE", "0")
    assert kernel_name(op, n_vec, mode) == "cheb_step_zmarch"
    z1 = per_probe(op, iv, degree, src, n_vec, mode)
    assert rel(z, z1) <= 1e-13
    # segmented z with a short ring
    monkeypatch.setenv("SDB_ZM_FUSE", "1")
    monkeypatch.setenv("SDB_ZM_NZS", "2")
    monkeypatch.setenv("SDB_ZM_R2", "4")
    z2 = per_probe(op, iv, degree, src, n_vec, mode)
    assert rel(z2, z1) <= 1e-13

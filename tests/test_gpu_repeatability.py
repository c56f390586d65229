"""Run-to-run bit-repeatability of the hand-synchronised kernels.

``compute-sanitizer`` is closed on this GPU pool, so racecheck /
synccheck cannot run.  What a shared-memory race, a missed mbarrier phase or a
ring slot released too early would produce is run-to-run variation: every
kernel here reduces in a fixed order and uses no floating-point atomics, so
repeated runs of the same workload must agree bit for bit.  Each family is run
several times, also with its shallowest ring (the tightest producer / consumer
hand-off); PDL chaining on against off is tests/test_gpu_pdl.py:

* ``cheb_step_zmarch``: TMA producer warp + mbarrier full/empty ring (7- and
  27-point grids, ring depths 3 and default);
* ``cheb_step_band``: cp.async gather rings, bulk-copy stage buffers and the
  yfar full/empty mbarrier pairs (ring depths 2 and default);
* Lanczos: the fused update+projection pass and the two-pass Gram schedule.
"""

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import _native
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.gpu

REPEATS = 5


def _moments(mat, iv, degree, kind, n_vec, mode):
    src = sdb.ProbeVectorSource(kind, seed=4, dim=mat.dim)
    run = E.run_chebyshev(sdb.apply_spectral_map(mat, iv), degree, src, n_vec, mode)
    return run.zeta_pp.cpu().numpy()


def _kernel(mat, n_vec, mode):
    from paper_1308_5467_b200.operators import device_matrix

    dm = device_matrix(mat, 0, E.stream_ptr(0))
    return _native.load().sdb_cheb_kernel(dm.handle, n_vec, mode).decode()


@pytest.mark.parametrize("shape", ["face7", "box27"])
@pytest.mark.parametrize("ring", [None, "3"])
def test_zmarch_ring_is_repeatable(monkeypatch, shape, ring):
    if ring:
        monkeypatch.setenv("SDB_ZM_R", ring)
    op = W.anderson_3d(32) if shape == "face7" else W.stencil27_3d(32)
    iv = W.gershgorin_interval(op)
    mode = _native.SDB_CHEB_DOUBLING
    assert "zmarch" in _kernel(op, 32, mode)
    first = _moments(op, iv, 60, "rademacher", 32, mode)
    assert np.all(np.isfinite(first))
    for _ in range(REPEATS - 1):
        np.testing.assert_array_equal(_moments(op, iv, 60, "rademacher", 32, mode), first)


@pytest.mark.parametrize("ring", [None, "2"])
@pytest.mark.parametrize("mode", ["doubling", "direct"])
def test_band_rings_are_repeatable(monkeypatch, ring, mode):
    if ring:
        monkeypatch.setenv("SDB_BAND_NB", ring)
    mat = W.dft_like(40_013)  # several tiles per block, ragged last tile
    iv = W.gershgorin_interval(mat)
    m = _native.SDB_CHEB_DOUBLING if mode == "doubling" else _native.SDB_CHEB_DIRECT
    assert "band" in _kernel(mat, 40, m)
    first = _moments(mat, iv, 50, "gaussian", 40, m)
    assert np.all(np.isfinite(first))
    for _ in range(REPEATS - 1):
        np.testing.assert_array_equal(_moments(mat, iv, 50, "gaussian", 40, m), first)


@pytest.mark.parametrize("gram", ["0", "1"])
def test_lanczos_passes_are_repeatable(monkeypatch, gram):
    monkeypatch.setenv("SDB_LZ_GRAM", gram)
    op = W.anderson_3d(16)
    src = sdb.ProbeVectorSource("gaussian", seed=2, dim=op.dim)
    v0 = src.draw(0)
    first = sdb.lanczos_factorize(op, v0, 60)
    for _ in range(REPEATS - 1):
        again = sdb.lanczos_factorize(op, v0, 60)
        np.testing.assert_array_equal(again.alpha, first.alpha)
        np.testing.assert_array_equal(again.beta, first.beta)

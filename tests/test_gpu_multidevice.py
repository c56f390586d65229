"""Single-process probe sharding: ``estimate_dos(..., devices=[...])``.

SURVEY 8(e) / §5: probe recurrences are independent units, so the drop-in
call can use several GPUs while keeping the reference's single-process
signature (compare.py:82-141, stochastic.py:64-74).  Only one GPU is visible
in this run, so the shards are placed on the same device (``devices=[0, 0]``:
two host threads, two streams, two workspaces); what is checked is the host
logic a multi-GPU box runs unchanged: contiguous shard ranges (even and
uneven), the probe-ordered gather on ``devices[0]``, the MATVEC credit, and
errors raised once, in probe order.  Per-probe rows agree with the unsharded
run to reduction-order rounding (the block partials of a probe depend on the
batch it runs in), the documented bound is 1e-13 relative.
"""

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import _native
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b))


@pytest.fixture(scope="module")
def anderson():
    op = W.anderson_3d(12)
    return op, W.gershgorin_interval(op)


@pytest.mark.parametrize("devices,n_vec", [([0], 8), ([0, 0], 8), ([0, 0, 0], 7), ([0, 0, 0, 0], 3)])
def test_per_probe_moments_in_probe_order(anderson, devices, n_vec):
    op, iv = anderson
    src = sdb.ProbeVectorSource("rademacher", seed=4, dim=op.dim)
    mapped = sdb.apply_spectral_map(op, iv)
    one = E.run_chebyshev(mapped, 80, src, n_vec, _native.SDB_CHEB_DOUBLING).zeta_pp.cpu().numpy()
    many = E.run_chebyshev(mapped, 80, src, n_vec, _native.SDB_CHEB_DOUBLING, device=devices)
    assert many.zeta_pp.device.index == 0
    got = many.zeta_pp.cpu().numpy()
    assert got.shape == one.shape
    for l in range(n_vec):  # row l is probe l whichever shard computed it
        assert rel(got[l], one[l]) <= 1e-13


@pytest.mark.parametrize("method,kw", [("kpm-jackson", {"product_formula": True}), ("kpm", {}), ("kpml", {}),
                                       ("lanczos", {"sigma": 0.3}), ("haydock", {}), ("cdos", {})])
def test_estimate_dos_devices_matches_single_device(anderson, method, kw):
    op, iv = anderson
    src = sdb.ProbeVectorSource("gaussian", seed=1, dim=op.dim)
    deg = 40 if method in ("lanczos", "haydock", "cdos") else 120
    a = sdb.estimate_dos(op, iv, method, deg, src, 9, grid_points=300, **kw)
    b = sdb.estimate_dos(op, iv, method, deg, src, 9, grid_points=300, devices=[0, 0], **kw)
    assert b.params["devices"] == [0, 0]
    assert a.params["matvec_count"] == b.params["matvec_count"]
    np.testing.assert_allclose(b.density, a.density, rtol=0, atol=1e-11 * max(1.0, np.max(np.abs(a.density))))
    if "moments" in a.params:
        assert rel(b.params["moments"], a.params["moments"]) <= 1e-13


def test_band_matrix_sharded(anderson):
    mat = W.dft_like(20_011)
    iv = W.gershgorin_interval(mat)
    src = sdb.ProbeVectorSource("gaussian", seed=2, dim=mat.dim)
    a = sdb.estimate_dos(mat, iv, "kpm-jackson", 100, src, 40, grid_points=200, product_formula=True)
    b = sdb.estimate_dos(mat, iv, "kpm-jackson", 100, src, 40, grid_points=200, product_formula=True,
                         devices=[0, 0, 0])
    assert rel(b.params["moments"], a.params["moments"]) <= 1e-13
    assert np.max(np.abs(a.density - b.density)) <= 1e-12


def test_user_counter_and_errors(anderson):
    op, iv = anderson
    counter = sdb.MatvecCounter(op)
    src = sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim)
    sdb.estimate_dos(counter, iv, "kpm", 30, src, 6, devices=[0, 0])
    assert counter.count == 6 * 30
    with pytest.raises(ValueError):
        sdb.estimate_dos(op, iv, "kpm", 30, src, 6, device=0, devices=[0])
    with pytest.raises(ValueError):
        sdb.estimate_dos(op, iv, "kpm", 30, src, 6, devices=[])

    class ZeroThird:
        dim = op.dim
        kind = "custom"

        def draw(self, i):
            return np.zeros(op.dim) if i == 2 else src.draw(i)

    with pytest.raises(ValueError, match="nonzero"):  # the reference's error, whichever shard holds probe 2
        sdb.estimate_dos(op, iv, "lanczos", 10, ZeroThird(), 5, sigma=0.5, devices=[0, 0])

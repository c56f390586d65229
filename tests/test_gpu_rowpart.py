"""Row-partitioned stencil moments on the GPU: z-ghost slab kernels, several
slabs driven in one process, halo planes pushed by the step kernels into the
neighbours' ghost planes (p2p: the same code path that writes peer-device
memory over NVLink when the slabs sit on several GPUs) or exchanged by device
copies.  The multi-rank NCCL exchange is covered on CPU (tests/test_rowpart_cpu.py)."""

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from oracle import specdens_oracle as O
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.rowpart import rowpartition_moments

pytestmark = pytest.mark.gpu


def generic_stencil():
    rng = np.random.default_rng(3)
    offs = [(1, 0, 0), (-1, 0, 0), (1, 1, 1), (-1, -1, -1), (0, 0, 1), (0, 0, -1)]
    return sdb.StencilOperator((6, 5, 8), offs, [0.3, 0.3, -0.2, -0.2, 0.5, 0.5], rng.uniform(-1, 1, 240))


@pytest.mark.parametrize("builder", [lambda: W.anderson_3d(8), lambda: W.stencil27_3d(7), generic_stencil],
                         ids=["face7", "box27", "generic"])
@pytest.mark.parametrize("n_slabs", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", [1, 0], ids=["doubling", "direct"])
@pytest.mark.parametrize("exchange", ["p2p", "copy"])
def test_slabs_match_oracle(builder, n_slabs, mode, exchange):
    op = builder()
    iv = W.gershgorin_interval(op)
    n_vec, deg = 20, 31
    src = sdb.ProbeVectorSource("rademacher", seed=4, dim=op.dim)
    got = rowpartition_moments(op, iv, deg, src, n_vec, mode=mode, n_slabs=n_slabs, exchange=exchange).cpu().numpy()
    ref = O.chebyshev_moments(op.csr, iv.center, iv.halfwidth, deg, "rademacher", 4, n_vec, mode="direct")
    assert np.max(np.abs(got - ref)) <= 1e-10 * np.max(np.abs(ref))


def test_slabs_match_unpartitioned_large():
    op = W.stencil27_3d(32)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim)
    whole = sdb.moments_via_product_formula(sdb.apply_spectral_map(op, iv), 60, src, 32)
    for n_slabs in (2, 8):
        for exchange in ("p2p", "copy"):
            got = rowpartition_moments(op, iv, 60, src, 32, n_slabs=n_slabs, exchange=exchange)
            got = got.mean(dim=0).cpu().numpy()
            assert np.max(np.abs(got - whole.zeta)) <= 1e-12 * np.max(np.abs(whole.zeta))


def test_p2p_devices_list_single_gpu():
    """The multi-device p2p driver (events between slab streams) with every
    slab on device 0: same moments as the single-device path."""
    op = W.anderson_3d(8)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=1, dim=op.dim)
    a = rowpartition_moments(op, iv, 21, src, 16, n_slabs=3, devices=[0, 0]).cpu().numpy()
    b = rowpartition_moments(op, iv, 21, src, 16, n_slabs=3, exchange="copy").cpu().numpy()
    np.testing.assert_array_equal(a, b)
    a = rowpartition_moments(op, iv, 21, src, 16, n_slabs=3, devices=[0, 0], layout="slabs").cpu().numpy()
    b = rowpartition_moments(op, iv, 21, src, 16, n_slabs=3, exchange="copy", layout="slabs").cpu().numpy()
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("mode", [1, 0], ids=["doubling", "direct"])
def test_boundary_interior_split_matches_whole_slab_steps(mode):
    """Copy exchange with the boundary / interior split (exchange on a second
    stream overlapping the interior planes) against whole-slab steps."""
    op = W.stencil27_3d(16)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=2, dim=op.dim)
    for n_slabs in (1, 2, 4):
        a = rowpartition_moments(op, iv, 41, src, 24, mode=mode, n_slabs=n_slabs, exchange="copy",
                                 overlap=True, layout="slabs").cpu().numpy()
        b = rowpartition_moments(op, iv, 41, src, 24, mode=mode, n_slabs=n_slabs, exchange="copy",
                                 overlap=False, layout="slabs").cpu().numpy()
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))


@pytest.mark.parametrize("builder", [lambda: W.anderson_3d(16), lambda: W.stencil27_3d(16)], ids=["face7", "box27"])
@pytest.mark.parametrize("n_slabs", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", [1, 0], ids=["doubling", "direct"])
@pytest.mark.parametrize("overlap", [True, False, "p2p"])
def test_plane_range_zmarch_slabs(builder, n_slabs, mode, overlap):
    """Row partition on full-size z-march blocks (sdb_cheb_step_planes): each
    slab computes its planes with the TMA z-march kernel; planes it does not
    own start as NaN, so a missing halo plane would poison the moments."""
    from paper_1308_5467_b200 import rowpart as RP

    op = builder()
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=6, dim=op.dim)
    plan = RP.SlabPlan(op.shape[2], n_slabs)
    assert isinstance(RP.make_slab(op, plan, 0, 32, 31, mode, 0, src, True), RP.PlaneSlab)
    if overlap == "p2p":  # halo pushed by the z-march epilogue into the neighbours' blocks
        got = rowpartition_moments(op, iv, 31, src, 32, mode=mode, n_slabs=n_slabs, exchange="p2p",
                                   layout="planes").cpu().numpy()
    else:
        got = rowpartition_moments(op, iv, 31, src, 32, mode=mode, n_slabs=n_slabs, exchange="copy",
                                   overlap=overlap, layout="planes").cpu().numpy()
    ref = O.chebyshev_moments(op.csr, iv.center, iv.halfwidth, 31, "rademacher", 6, 32, mode="direct")
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - ref)) <= 1e-10 * np.max(np.abs(ref))


def test_plane_range_matches_unpartitioned_large():
    op = W.stencil27_3d(32)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim)
    whole = sdb.moments_via_product_formula(sdb.apply_spectral_map(op, iv), 60, src, 32)
    for n_slabs in (2, 8):
        got = rowpartition_moments(op, iv, 60, src, 32, n_slabs=n_slabs, exchange="copy", layout="planes")
        got = got.mean(dim=0).cpu().numpy()
        assert np.max(np.abs(got - whole.zeta)) <= 1e-12 * np.max(np.abs(whole.zeta))

"""Row-partitioned (z-slab) recurrence: host driver and halo exchange on CPU.

The per-slab compute is tests/slab_reference.NumpySlab (a NumPy restatement of
the step kernel on ghosted slabs); the driver, plan and halo exchange are the
product code in paper_1308_5467_b200/rowpart.py.  Multi-rank: gloo, world 2.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import specdens_oracle as O
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.rowpart import SlabPlan, run_rowpartition

DEG = 23


def reference(op, n_vec, doubling):
    iv = W.gershgorin_interval(op)
    per = O.chebyshev_moments(op.csr, iv.center, iv.halfwidth, DEG, "rademacher", 4, n_vec,
                              mode="doubling" if doubling else "direct")
    return per, iv


def probes(op, n_vec):
    return np.array([O.draw_probe("rademacher", 4, op.dim, l) for l in range(n_vec)])


@pytest.mark.parametrize("n_slabs", [1, 2, 3, 5])
@pytest.mark.parametrize("doubling", [True, False])
@pytest.mark.parametrize("overlap", [True, False])
def test_single_process_slabs(n_slabs, doubling, overlap):
    from tests.slab_reference import NumpySlab, fill_probes

    op = W.stencil27_3d(6) if n_slabs % 2 else W.anderson_3d(7)
    n_vec = 3
    ref, iv = reference(op, n_vec, doubling)
    plan = SlabPlan(op.shape[2], n_slabs)
    pr = probes(op, n_vec)
    slabs = [NumpySlab(op, plan, s, n_vec, DEG, doubling) for s in range(n_slabs)]
    for sl in slabs:
        fill_probes(sl, pr, op.shape)
    got = run_rowpartition(slabs, plan, iv.center, iv.halfwidth, DEG, 1 if doubling else 0, overlap=overlap).numpy()
    assert all(sl.parts for sl in slabs) == (op.shape[2] // n_slabs >= 3)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, overlap, planes=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.slab_reference import NumpyPlaneSlab, NumpySlab, fill_plane_probes, fill_probes

        op = W.anderson_3d(6)
        n_vec = 2
        iv = W.gershgorin_interval(op)
        plan = SlabPlan(op.shape[2], world)
        if planes:
            sl = NumpyPlaneSlab(op, plan, rank, n_vec, DEG, True)
            fill_plane_probes(sl, probes(op, n_vec))
        else:
            sl = NumpySlab(op, plan, rank, n_vec, DEG, True)
            fill_probes(sl, probes(op, n_vec), op.shape)
        assert sl.parts  # 3 planes per slab: the boundary / interior split applies
        got = run_rowpartition([sl], plan, iv.center, iv.halfwidth, DEG, 1, group=None,
                               rank_of_slab=lambda s: s, overlap=overlap)
        q.put((rank, got.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("planes", [False, True], ids=["slab-blocks", "full-blocks"])
def test_two_rank_halo_exchange_gloo(overlap, planes):
    import sys

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, overlap, planes)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    op = W.anderson_3d(6)
    ref, _ = reference(op, 2, True)
    for r in (0, 1):
        assert np.max(np.abs(res[r] - ref)) <= 1e-11 * np.max(np.abs(ref))
    np.testing.assert_array_equal(res[0], res[1])


@pytest.mark.parametrize("n_slabs", [1, 2, 3, 5])
@pytest.mark.parametrize("doubling", [True, False])
@pytest.mark.parametrize("overlap", [True, False])
def test_single_process_full_blocks(n_slabs, doubling, overlap):
    """The plane-range driver (PlaneSlab layout: full-size blocks, global plane
    indices in the exchange) with NaN outside what each slab may read."""
    from tests.slab_reference import NumpyPlaneSlab, fill_plane_probes

    op = W.stencil27_3d(6) if n_slabs % 2 else W.anderson_3d(7)
    n_vec = 3
    ref, iv = reference(op, n_vec, doubling)
    plan = SlabPlan(op.shape[2], n_slabs)
    pr = probes(op, n_vec)
    slabs = [NumpyPlaneSlab(op, plan, s, n_vec, DEG, doubling) for s in range(n_slabs)]
    for sl in slabs:
        fill_plane_probes(sl, pr)
    got = run_rowpartition(slabs, plan, iv.center, iv.halfwidth, DEG, 1 if doubling else 0, overlap=overlap).numpy()
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))

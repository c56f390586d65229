"""Multi-GPU front doors on one GPU: a world-size-1 NCCL group exercises the
probe-shard gather and the row-partition all-reduce code paths for real."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_1308_5467_b200 as sdb
from oracle import specdens_oracle as O
from paper_1308_5467_b200 import distributed as D
from paper_1308_5467_b200 import workloads as W
from paper_1308_5467_b200.rowpart import rowpartition_moments

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    if dist.is_initialized():
        yield None
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield None
    dist.destroy_process_group()


@pytest.mark.parametrize("method", ["kpm-jackson", "kpm", "spectroscopic", "delta-cheb", "kpml", "dgl", "lanczos",
                                    "haydock", "cdos"])
def test_sharded_estimate_matches_single(nccl_group, method):
    op = W.anderson_3d(10)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("gaussian", seed=3, dim=op.dim)
    kw = {"kpm-jackson": {"product_formula": True}, "spectroscopic": {"product_formula": True},
          "lanczos": {"sigma": 0.05}, "dgl": {"sigma": 0.2}, "haydock": {"eta": 0.1}}.get(method, {})
    deg = 30 if method in ("lanczos", "haydock", "cdos") else 61
    one = sdb.estimate_dos(op, iv, method, deg, src, 7, grid_points=300, **kw)
    sh = D.estimate_dos_sharded(op, iv, method, deg, src, 7, grid_points=300, **kw)
    np.testing.assert_allclose(sh.density, one.density, rtol=0, atol=1e-13)
    assert sh.params["matvec_count"] == one.params["matvec_count"]


def test_rowpartition_with_group(nccl_group):
    op = W.stencil27_3d(8)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=1, dim=op.dim)
    got = rowpartition_moments(op, iv, 25, src, 12, group=dist.group.WORLD).cpu().numpy()
    ref = O.chebyshev_moments(op.csr, iv.center, iv.halfwidth, 25, "rademacher", 1, 12, mode="direct")
    assert np.max(np.abs(got - ref)) <= 1e-10 * np.max(np.abs(ref))

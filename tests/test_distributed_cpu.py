"""N > 1 logic of the probe-shard path on CPU (gloo, world_size 2).

The GPU path (paper_1308_5467_b200/distributed.py) shards the probe indices
into contiguous ranges, runs each range's recurrences on its rank and
all-gathers the per-probe rows once.  Here the per-rank compute is the CPU
oracle (test infrastructure), so the test checks exactly the host logic: the
shard ranges, the padded all-gather for uneven shards, and that the
probe-ordered assembly gives the single-process result bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1308_5467_b200.distributed import gather_probe_rows, shard_range


def test_shard_ranges_partition_probes():
    for n_vec in (1, 2, 7, 64, 129):
        for world in (1, 2, 3, 8):
            if n_vec < world:
                continue
            ranges = [shard_range(n_vec, world, r) for r in range(world)]
            assert ranges[0][0] == 0
            for (s0, c0), (s1, _) in zip(ranges, ranges[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in ranges) == n_vec
            assert max(c for _, c in ranges) - min(c for _, c in ranges) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_vec, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import specdens_oracle as O
        from paper_1308_5467_b200 import workloads as W

        op = W.anderson_3d(6)
        iv = W.gershgorin_interval(op)
        start, count = shard_range(n_vec, world, rank)
        per = O.chebyshev_moments(op.csr, iv.center, iv.halfwidth, 30, "rademacher", 0, count, mode="doubling",
                                  indices=range(start, start + count))
        rows = gather_probe_rows(torch.from_numpy(per), n_vec)
        zeta = O.average_moments(rows.numpy())
        out_q.put((rank, rows.numpy(), zeta))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_vec", [6, 7])  # even and uneven shards
def test_probe_shard_gather_matches_single_process(n_vec):
    from oracle import specdens_oracle as O
    from paper_1308_5467_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_vec, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    op = W.anderson_3d(6)
    iv = W.gershgorin_interval(op)
    ref = O.chebyshev_moments(op.csr, iv.center, iv.halfwidth, 30, "rademacher", 0, n_vec, mode="doubling")
    for _, rows, zeta in results:
        np.testing.assert_array_equal(rows, ref)  # probe order preserved
        np.testing.assert_array_equal(zeta, O.average_moments(ref))  # GPU-count independent


def _raise_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1308_5467_b200 as sdb
        from paper_1308_5467_b200 import workloads as W
        from paper_1308_5467_b200.distributed import estimate_dos_sharded

        op = W.anderson_3d(4)
        iv = W.gershgorin_interval(op)
        src = sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim)
        try:
            estimate_dos_sharded(op, iv, "kpm-jackson", 10, src, 1)  # one probe, two ranks
            out_q.put((rank, "no error"))
        except ValueError as exc:
            out_q.put((rank, str(exc)))
        dist.barrier()  # both ranks are still in step: nobody is stuck in a gather
    finally:
        dist.destroy_process_group()


def test_fewer_probes_than_ranks_raises_on_every_rank():
    """A rank without probes must not raise alone while its peers wait in the
    all-gather: the check depends only on the arguments, so all ranks raise."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_raise_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert set(results) == {0, 1}
    for msg in results.values():
        assert "at least one probe" in msg

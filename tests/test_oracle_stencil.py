"""Pin the C oracle's stencil path (used for C5 at 256^3, where the CSR would
be 5.4 GB of host arrays) against its CSR path on the stencil's own CSR.

The CSR path is itself pinned bit-for-bit to the reference (test_oracle_golden);
the stencil path sums an interior row's terms in the same (sorted-column)
order, so only rows on the periodic faces can differ, by rounding.
"""

import numpy as np
import pytest

import paper_1308_5467_b200 as sdb
from oracle import c_oracle
from paper_1308_5467_b200 import workloads as W

pytestmark = pytest.mark.skipif(not c_oracle.available(), reason="oracle/build/liboracle.so not built")


def rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


@pytest.mark.parametrize("L", [24, 32])
@pytest.mark.parametrize("mode", ["doubling", "direct"])
def test_stencil27_oracle_matches_csr_oracle(L, mode):
    op = W.stencil27_3d(L)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim)
    probes = np.array([src.draw(l) for l in range(2)])
    st = c_oracle.stencil_moments(op, iv.center, iv.halfwidth, 60, probes, mode=mode, threads=2)
    cs = c_oracle.cheb_moments(op.csr, iv.center, iv.halfwidth, 60, probes, mode=mode, threads=2)
    assert rel(st, cs) <= 1e-12


def test_face7_oracle_matches_csr_oracle():
    op = W.anderson_3d(16)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("gaussian", seed=1, dim=op.dim)
    probes = np.array([src.draw(l) for l in range(3)])
    st = c_oracle.stencil_moments(op, iv.center, iv.halfwidth, 41, probes, threads=3)
    cs = c_oracle.cheb_moments(op.csr, iv.center, iv.halfwidth, 41, probes, threads=3)
    assert rel(st, cs) <= 1e-12

"""Programmatic dependent launch between recurrence steps changes scheduling only.

Every step kernel waits (griddepcontrol.wait) before touching global memory,
so chaining the steps with PDL must give bit-identical moments to plain
stream-ordered launches (SDB_PDL=0; read once per process, hence the
subprocesses).  Covers the CSR kernel (C1), the z-march kernel (7- and
27-point grids), the row-panel grid kernel and the fused-pair z-march.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import workloads as W
out = {}
cases = {
    "c1_csr": (W.build_matrix("C1"), "gaussian", 20, 100),
    "c3_csr": (W.dft_like(20000, n_random=10, seed=3), "gaussian", 24, 30),
    "face7": (W.anderson_3d(24), "rademacher", 16, 60),
    "box27": (W.stencil27_3d(16), "rademacher", 8, 41),
}
for name, (op, kind, nv, deg) in cases.items():
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource(kind, seed=0, dim=op.dim)
    for pf in (False, True):
        m = (sdb.moments_via_product_formula if pf else sdb.compute_chebyshev_moments)(
            sdb.apply_spectral_map(op, iv), deg, src, nv)
        out[f"{name}_{int(pf)}"] = m.zeta
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, pdl, extra_env=None):
    path = tmp_path / f"pdl{pdl}_{'x' if extra_env else 'd'}.npz"
    env = dict(os.environ, SDB_PDL=str(pdl), **(extra_env or {}))
    subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(path)], check=True, env=env, timeout=600)
    return np.load(path)


@pytest.mark.parametrize("extra_env", [None, {"SDB_ZMARCH": "0"}, {"SDB_ZM_FUSE": "1"}],
                         ids=["default", "row-panel", "fused-pairs"])
def test_pdl_chaining_is_bit_identical(tmp_path, extra_env):
    on = _run(tmp_path, 1, extra_env)
    off = _run(tmp_path, 0, extra_env)
    assert sorted(on.files) == sorted(off.files)
    for k in on.files:
        np.testing.assert_array_equal(on[k], off[k], err_msg=k)

"""Small fused z-march run for compute-sanitizer / debugging."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1308_5467_b200 as sdb  # noqa: E402
from paper_1308_5467_b200 import _native  # noqa: E402
from paper_1308_5467_b200 import engine as E  # noqa: E402
from tests.test_gpu_zmarch import make_stencil  # noqa: E402
from oracle import specdens_oracle as O  # noqa: E402
from paper_1308_5467_b200 import workloads as W  # noqa: E402

shape = tuple(int(v) for v in os.environ.get("SHAPE", "8,8,5").split(","))
kind = os.environ.get("KIND", "face7")
n_vec = int(os.environ.get("NVEC", "8"))
degree = int(os.environ.get("DEG", "5"))
op = make_stencil(shape, kind, seed=1)
iv = W.gershgorin_interval(op)
src = sdb.ProbeVectorSource("gaussian", seed=1, dim=op.dim)
run = E.run_chebyshev(sdb.apply_spectral_map(op, iv), degree, src, n_vec, _native.SDB_CHEB_DOUBLING)
z = run.zeta_pp.cpu().numpy()
ref = np.array(O.chebyshev_moments(op, iv.center, iv.halfwidth, degree, "gaussian", 1, n_vec, mode="doubling"))
print("rel", np.max(np.abs(z - ref)) / np.max(np.abs(ref)))
print(z[0], ref[0])

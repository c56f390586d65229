"""Host-side profile of one COLD C3 estimate (fresh matrix object, fresh probe source)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import workloads as W

cfg = W.CONFIGS["C3"]
op = W.build_matrix("C3")
iv = W.gershgorin_interval(op)
warm_src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=op.dim)
sdb.estimate_dos(op, iv, "kpm-jackson", 20, warm_src, 8, grid_points=100, product_formula=True)  # context, kernels
torch.cuda.synchronize()
for rep in range(2):
    cold_op = sdb.SparseSymmetricMatrix(csr=op.csr)
    cold_src = sdb.ProbeVectorSource(cfg.probe_kind, seed=rep + 1, dim=op.dim)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    sdb.estimate_dos(cold_op, iv, "kpm-jackson", cfg.degree, cold_src, cfg.n_vec, grid_points=cfg.grid_points,
                     product_formula=True)
    pr.disable()
    print("cold call ms", (time.perf_counter() - t0) * 1e3)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
    del cold_op, cold_src

"""C1 moment run (resident kernel) timed by CUDA events, warm (no L2 flush between runs) and cold
(256 MB write before each): the difference is the cold start of a kernel that runs once."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch

import paper_1308_5467_b200 as sdb
from paper_1308_5467_b200 import _native
from paper_1308_5467_b200 import engine as E
from paper_1308_5467_b200 import workloads as W

cfg = W.CONFIGS["C1"]
op = W.build_matrix("C1")
iv = W.gershgorin_interval(op)
src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=op.dim)
probes = src.draw_block(0, cfg.n_vec).to(0)
mapped = sdb.apply_spectral_map(op, iv)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=0)
for label, do_flush in (("warm", False), ("cold", True), ("warm", False)):
    ts = []
    for _ in range(8):
        if do_flush:
            flush.fill_(1)
        torch.cuda.synchronize()
        run = E.run_chebyshev(mapped, cfg.degree, None, cfg.n_vec, _native.SDB_CHEB_DOUBLING, device=0, probes=probes,
                              time_steps=True)
        torch.cuda.synchronize()
        ts.append(run.step_ms * 1e3)
    print(label, "us per moment run:", " ".join(f"{t:.1f}" for t in ts), flush=True)

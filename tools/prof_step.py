"""Run a short KPM moment run on one config for ncu captures of the step kernel.

  python tools/prof_step.py C2 [degree]     (env vars select kernels / tiles)
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1308_5467_b200 as sdb
    from paper_1308_5467_b200 import _native
    from paper_1308_5467_b200 import engine as E
    from paper_1308_5467_b200 import workloads as W

    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    degree = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = W.CONFIGS[name]
    op = W.build_matrix(name)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=op.dim)
    probes = src.draw_block(0, cfg.n_vec).to(0)
    run = E.run_chebyshev(sdb.apply_spectral_map(op, iv), degree, None, cfg.n_vec, _native.SDB_CHEB_DOUBLING,
                          device=0, probes=probes, time_steps=True)
    torch.cuda.synchronize()
    print(name, "step ms total", run.step_ms)


if __name__ == "__main__":
    main()

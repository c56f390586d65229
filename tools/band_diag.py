"""Time the C3 band + far step kernel under its diagnostic switches (one process,
matrix built once):  python tools/band_diag.py [degree] [VAR=VAL,VAR=VAL ...]"""
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

    degree = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    variants = sys.argv[2:] or ["", "SDB_BAND_DIAG=4", "SDB_BAND_DIAG=8", "SDB_BAND_DIAG=12", "SDB_BAND_DIAG=16",
                                "SDB_BAND_NB=2", "SDB_BAND=0"]
    cfg = W.CONFIGS["C3"]
    op = W.build_matrix("C3")
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=op.dim)
    probes = src.draw_block(0, cfg.n_vec).to(0)
    mapped = sdb.apply_spectral_map(op, iv)
    steps = (degree + 1) // 2
    for v in variants:
        sets = [kv.split("=") for kv in v.split(",") if kv]
        for k, val in sets:
            os.environ[k] = val
        best = 1e30
        for _ in range(3):
            run = E.run_chebyshev(mapped, degree, None, cfg.n_vec, _native.SDB_CHEB_DOUBLING, device=0, probes=probes,
                                  time_steps=True)
            torch.cuda.synchronize()
            best = min(best, run.step_ms)
        print(f"{v or 'default':40s} {best / steps * 1e3:9.1f} us/step", flush=True)
        for k, _ in sets:
            os.environ.pop(k, None)


if __name__ == "__main__":
    main()

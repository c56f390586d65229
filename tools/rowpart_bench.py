"""Time the row-partitioned recurrence on one GPU (slabs in one process).

  python tools/rowpart_bench.py [--n 128] [--slabs 2] [--degree 200] [--n-vec 32]

Prints ms per recurrence step for: the unpartitioned estimate (z-march), the
p2p epilogue push, and the copy exchange with / without the boundary /
interior split.  One GPU only: the exchange is a device copy, so this measures
the split's own cost, not NVLink overlap.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--slabs", type=int, default=2)
    ap.add_argument("--degree", type=int, default=200)
    ap.add_argument("--n-vec", type=int, default=32)
    args = ap.parse_args()
    import torch

    import paper_1308_5467_b200 as sdb
    from paper_1308_5467_b200 import workloads as W
    from paper_1308_5467_b200.rowpart import rowpartition_moments

    op = W.stencil27_3d(args.n)
    iv = W.gershgorin_interval(op)
    src = sdb.ProbeVectorSource("rademacher", seed=0, dim=op.dim)
    steps = (args.degree + 1) // 2

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) * 1e3 / steps

    import paper_1308_5467_b200.rowpart as RP
    from paper_1308_5467_b200 import _native

    mode = _native.SDB_CHEB_DOUBLING
    res = {"whole": timed(lambda: sdb.moments_via_product_formula(sdb.apply_spectral_map(op, iv), args.degree,
                                                                  src, args.n_vec))}
    plan = RP.SlabPlan(op.shape[2], args.slabs)
    slabs = []
    for s in range(args.slabs):  # probes staged once (host Philox draws are not the step)
        sl = RP.DeviceSlab(op, plan, s, args.n_vec, args.degree, mode, 0)
        RP.ghosted_probe_block(src, 0, args.n_vec, op.shape, sl.z0, sl.nzl, sl.ldv, sl.blocks[0])
        slabs.append(sl)
    c, d = float(iv.center), float(iv.halfwidth)
    res["p2p"] = timed(lambda: RP.run_rowpartition_p2p(slabs, plan, c, d, args.degree, mode))
    res["copy"] = timed(lambda: RP.run_rowpartition(slabs, plan, c, d, args.degree, mode, overlap=False))
    res["copy+split"] = timed(lambda: RP.run_rowpartition(slabs, plan, c, d, args.degree, mode, overlap=True))
    pslabs = [RP.make_slab(op, plan, s, args.n_vec, args.degree, mode, 0, src, True) for s in range(args.slabs)]
    res["planes"] = timed(lambda: RP.run_rowpartition(pslabs, plan, c, d, args.degree, mode, overlap=False))
    res["planes+split"] = timed(lambda: RP.run_rowpartition(pslabs, plan, c, d, args.degree, mode, overlap=True))
    res["planes+p2p"] = timed(lambda: RP.run_rowpartition_p2p(pslabs, plan, c, d, args.degree, mode))
    print({k: round(v, 3) for k, v in res.items()}, f"ms/step (n={args.n}^3, {args.slabs} slabs, "
          f"{args.n_vec} probes; 'whole' includes its probe draw)")


if __name__ == "__main__":
    main()

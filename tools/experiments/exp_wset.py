"""How the C3 step scales with the gathered working set: the same matrix class at n = 250k .. 1M
(16-probe slice = n x 128 B), us per step and ns per row."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1308_5467_b200 as sdb
    from paper_1308_5467_b200 import _native
    from paper_1308_5467_b200 import engine as E
    from paper_1308_5467_b200 import workloads as W

    sizes = [int(a) for a in sys.argv[1:] if a.isdigit()] or [250_000, 500_000, 750_000, 1_000_000]
    variants = [a for a in sys.argv[1:] if not a.isdigit()] or [""]
    for n in sizes:
        op = W.dft_like(n)
        iv = W.gershgorin_interval(op)
        src = sdb.ProbeVectorSource("gaussian", seed=0, dim=op.dim)
        probes = src.draw_block(0, 128).to(0)
        mapped = sdb.apply_spectral_map(op, iv)
        for v in variants:
            sets = [kv.split("=") for kv in v.split(",") if kv]
            for k, val in sets:
                os.environ[k] = val
            best = 1e30
            for _ in range(3):
                run = E.run_chebyshev(mapped, 100, None, 128, _native.SDB_CHEB_DOUBLING, device=0, probes=probes,
                                      time_steps=True)
                torch.cuda.synchronize()
                best = min(best, run.step_ms)
            us = best / 50 * 1e3
            print(f"n={n:8d} slice={n * 128 / 2**20:6.1f} MB  {v or 'default':36s} {us:8.1f} us/step  "
                  f"{us * 1e3 / n:6.3f} ns/row", flush=True)
            for k, _ in sets:
                os.environ.pop(k, None)
        del op, mapped, probes
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

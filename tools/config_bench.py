"""Time every BASELINE config on one GPU (device-resident probes, CUDA events).

  python tools/config_bench.py [C1 C2 C3 C4 C5] [--format csr|stencil] [--reps 3] [--cpu]

Prints one JSON line per config: wall time of one full estimate, GNNZ-vec/s
(nnz * n_vec * M / t), the step-kernel roofline fraction (KPM) or the whole
Lanczos run's algorithmic-bytes rate (Lanczos).  With --cpu every line also
carries the CPU baseline timed on this box's host cores (BASELINE.md §2,
SURVEY §8d): the C restatement of the reference recurrence on all host
threads for the KPM configs (C5 through its stencil path), the NumPy/SciPy
restatement of ``lanczos_dos`` for C4 -- bounded samples (a few probes,
reduced M), extrapolated linearly in probes x steps and labelled so.  Not the
headline bench (bench.py measures C3); used for DESIGN.md and profiles/.
"""

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cpu_baseline(name, cfg, op, iv, nnz, gpu_seconds, target_s):
    """Bounded CPU sample of the config's hot path on this box, extrapolated to the full config."""
    import numpy as np

    import bench as B
    from oracle import c_oracle as C
    from oracle import specdens_oracle as O

    threads = B.cpu_threads()
    base = {"cores": threads, "cpu_model": B.cpu_model(), "kind": "port", "extrapolated": True}
    if cfg.method == "lanczos":
        # lanczos_dos(A, iv, 100, source, n_vec, sigma, grid) of the NumPy/SciPy restatement
        # (lanczos.py:198-219); OpenBLAS threading left at its default
        import paper_1308_5467_b200 as sdb

        grid = sdb.interval_grid(iv, cfg.grid_points)
        sample = 2
        t0 = time.perf_counter()
        O.lanczos_dos(op.csr, cfg.degree, cfg.probe_kind, 0, sample, cfg.sigma, grid)
        secs = time.perf_counter() - t0
        full = secs * cfg.n_vec / sample
        return dict(base, seconds_full_config_extrapolated=full, gpu_speedup=full / gpu_seconds,
                    sample=f"{name}: lanczos_dos with {sample} of {cfg.n_vec} probes, m={cfg.degree} steps, full "
                           f"reorthogonalisation (oracle/specdens_oracle.py, NumPy/SciPy, default BLAS threads): "
                           f"{secs:.2f} s; time ~ probes")
    if hasattr(op, "offsets"):  # stencil operator (C5, C2 as generated): the C oracle's stencil path
        probes = min(cfg.n_vec, threads)
        pr = np.array([O.draw_probe(cfg.probe_kind, 0, op.dim, l) for l in range(probes)])

        def run(deg):
            t0 = time.perf_counter()
            C.stencil_moments(op, iv.center, iv.halfwidth, deg, pr, mode="doubling", threads=threads)
            return time.perf_counter() - t0

        cal = run(4)
        deg = max(4, min(cfg.degree, int(target_s / (cal / 4)) // 2 * 2))
        secs = run(deg)
        rate = nnz * probes * deg / secs / 1e9
    else:
        sm = B.CpuSampler(op, iv, cfg, True, 0, target_s)
        secs = sm.sample()
        probes, deg, rate = sm.probes, sm.degree, sm.rate(secs)
    full = nnz * cfg.n_vec * cfg.degree / rate / 1e9
    return dict(base, value=rate, unit="GNNZ-vec/s", cores=min(threads, probes),
                seconds_full_config_extrapolated=full, gpu_speedup=full / gpu_seconds,
                sample=f"{name}: {probes} of {cfg.n_vec} probes x M={deg} of {cfg.degree} (doubling), C restatement "
                       f"of the reference recurrence (oracle/c), one probe per pthread: {secs:.2f} s; rate of the "
                       "truncated run = extrapolated full-config rate (time ~ steps x probes)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--format", default="native", choices=["native", "csr", "csr-raw"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu", action="store_true", help="time the CPU oracle beside each config (bounded sample)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="target wall time of one CPU sample")
    args = ap.parse_args()
    if args.format == "csr-raw":
        os.environ["SDB_AUTO_STENCIL"] = "0"
    import torch

    import paper_1308_5467_b200 as sdb
    from paper_1308_5467_b200 import _native
    from paper_1308_5467_b200 import engine as E
    from paper_1308_5467_b200 import lanczos as LZ
    from paper_1308_5467_b200 import workloads as W

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    dev = 0
    torch.cuda.set_device(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for name in args.configs:
        cfg = W.CONFIGS[name]
        t0 = time.time()
        op = W.build_matrix(name)
        iv = W.gershgorin_interval(op)
        if args.format != "native" and not isinstance(op, sdb.SparseSymmetricMatrix):
            op = sdb.SparseSymmetricMatrix(csr=op.csr)
        gen_s = time.time() - t0
        n = op.dim
        nnz = int(op.csr.nnz) if isinstance(op, sdb.SparseSymmetricMatrix) else int(op.nnz)
        src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=n)
        probes = src.draw_block(0, cfg.n_vec).to(dev)
        times, kms = [], []
        if cfg.method == "lanczos":
            grid = E.to_device(sdb.interval_grid(iv, cfg.grid_points), dev)
            for r in range(args.reps + 1):
                flush.fill_(1)
                torch.cuda.synchronize()
                t = time.perf_counter()
                res, theta, tau2, sd, _ = LZ.lanczos_quadrature_device(op, cfg.degree, None, cfg.n_vec,
                                                                       device=dev, probes=probes)
                stream = E.stream_ptr(dev)
                nodes, weights = LZ._pool_device(theta, tau2, sd, cfg.n_vec, dev, stream)
                LZ._blur_device(nodes, weights, grid, "gaussian", cfg.sigma, 1.0, dev, stream)
                torch.cuda.synchronize()
                if r:
                    times.append(time.perf_counter() - t)
            dm = res.base
            ldv = E.block_ldv(cfg.n_vec)
            from paper_1308_5467_b200.operators import device_matrix

            ma = device_matrix(res.base, dev, E.stream_ptr(dev)).bytes_per_pass
            m = cfg.degree
            # traffic of the schedule that ran.  Two-pass Gram-corrected CGS2 (default for
            # n >= 16384, steps <= n / 64): SpMM 4 block passes + proj (V, w, v_j) + update (V, w rmw);
            # fused three-pass (SDB_LZ_GRAM=0): SpMM 4 + proj (V, w) + K5c (V, w in, w out) +
            # update (V, w rmw); SDB_LZ_FUSED=0 as well: the 4-pass reference order
            genv = os.environ.get("SDB_LZ_GRAM", "")
            gram = genv == "1" or (genv != "0" and n >= 16384 and m <= n // 64)
            fused = os.environ.get("SDB_LZ_FUSED", "1") != "0" and m <= 256
            per_step = (lambda j: 2 * (j + 1) + 8) if gram else (
                (lambda j: 3 * (j + 1) + 9) if fused else (lambda j: 4 * (j + 1) + 11))
            passes = 2 if gram else 3
            total = sum(ma + 8 * n * ldv * per_step(j) for j in range(m))
            minimal = sum(ma + 8 * n * ldv * (passes * (j + 1) + 3) for j in range(m))
            minimal3 = sum(ma + 8 * n * ldv * (3 * (j + 1) + 3) for j in range(m))
            t = statistics.median(times)
            out = {"config": name, "method": "lanczos", "n": n, "nnz": nnz, "n_vec": cfg.n_vec, "steps": m,
                   "seconds": t, "gnnz_vec_s": nnz * cfg.n_vec * m / t / 1e9,
                   "schedule": ("two-pass Gram-corrected CGS2 (2 basis reads)" if gram else
                                "fused CGS2 (3 basis reads)" if fused else "4-pass CGS2"),
                   "bytes_moved_model_TB": total / 1e12, "achieved_GBs": total / t / 1e9,
                   "frac_of_peak": total / t / 1e9 / peak, "minimal_TB": minimal / 1e12,
                   "frac_vs_minimal_bytes": minimal / t / 1e9 / peak,
                   "minimal_3pass_TB": minimal3 / 1e12, "frac_vs_minimal_3pass_bytes": minimal3 / t / 1e9 / peak,
                   "gen_s": gen_s}
        else:
            mode = _native.SDB_CHEB_DOUBLING
            mapped = sdb.apply_spectral_map(op, iv)
            grid = sdb.unit_grid(cfg.grid_points)
            from paper_1308_5467_b200.compare import kpm_dos_device

            for r in range(args.reps + 1):
                flush.fill_(1)
                torch.cuda.synchronize()
                t = time.perf_counter()
                zeta, vals, dens, nonfinite, run = kpm_dos_device(mapped, cfg.degree, None, cfg.n_vec, "jackson",
                                                                  grid, True, device=dev, probes=probes,
                                                                  time_steps=True)
                torch.cuda.synchronize()
                if r:
                    times.append(time.perf_counter() - t)
                    kms.append(run.step_ms)
            t = statistics.median(times)
            steps = (cfg.degree + 1) // 2
            bytes_launch = run.dm.bytes_per_pass + 24 * n * cfg.n_vec
            k = statistics.median(kms) * 1e-3
            out = {"config": name, "method": "kpm-jackson (doubling)", "n": n, "nnz": nnz, "n_vec": cfg.n_vec,
                   "degree": cfg.degree, "format": "stencil" if run.dm.format == _native.SDB_FMT_STENCIL else "csr",
                   "detected_stencil": run.dm.detected_stencil, "seconds": t,
                   "gnnz_vec_s": nnz * cfg.n_vec * cfg.degree / t / 1e9,
                   "step_us": k / steps * 1e6, "bytes_per_step": bytes_launch,
                   "achieved_GBs": bytes_launch / (k / steps) / 1e9,
                   "frac_of_peak": bytes_launch / (k / steps) / 1e9 / peak, "nonfinite": bool(nonfinite),
                   "gen_s": gen_s}
        if args.cpu:
            try:
                out["cpu_baseline"] = cpu_baseline(name, cfg, op, iv, nnz, out["seconds"], args.cpu_seconds)
            except Exception as exc:  # the baseline must not sink the GPU line
                out["cpu_baseline"] = {"failed": repr(exc)}
        print(json.dumps(out), flush=True)
        del op, probes
        E.Workspace.release()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

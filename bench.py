"""Benchmark: stochastic Chebyshev-moment KPM DOS on the GPU (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--config C2] [--impl reference]

One "step" is one full KPM estimate of the config: all probes' moments (the
fused recurrence), probe mean, Jackson coefficients and the DOS on the grid.
Default workload: config 3, the one BASELINE.json's metric is quoted on
("sharded by probe vector across 1/2/4/8 GPUs"): synthetic DFT-like matrix,
n = 1e6, ~61 nnz/row (band of half-width 20 + ~20 random off-band entries per
row), fp64 CSR, KPM M = 1000, 128 Gaussian probes, Jackson damping, 2000 DOS
points, product-formula (doubling) moments: 500 SpMM steps deliver the 1001
moments.  --config C1 | C2 | C5 select the other KPM configs.

Metric: GNNZ-vec/s = nnz * n_vec * M / t (M = moments delivered).  ``value``
is measured with the matrix and the probes resident in HBM (L2 flushed
between steps); ``e2e`` goes through the public ``estimate_dos`` with the
probes in pinned host memory, copied host->device every step, and the moments
and density read back every step.  Multi-GPU (torchrun): probe sharding,
STRONG scaling -- the config's n_vec probes are split into contiguous ranges,
rank r runs shard_range(n_vec, N, r), the per-probe moments are all-gathered
once per step (the only collective) and averaged in probe order (C5: row
partition, also strong).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--format", default="csr", choices=["csr", "csr-raw", "stencil"],
                    help="csr: the config's CSR matrix through the matrix layer (stencil detection on); "
                         "csr-raw: CSR kernel forced; stencil: StencilOperator input")
    ap.add_argument("--direct", action="store_true", help="direct (non-doubling) moments")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-probes", type=int, default=0)
    ap.add_argument("--cpu-sample-seconds", type=float, default=0.0,
                    help="target wall time of one CPU sample (default: 12 s for cpu_baseline, 4 s per "
                         "reference-arm step)")
    ap.add_argument("--no-cold", action="store_true", help="skip the cold first-call e2e measurement")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_traffic(config, fmt, kernel):
    """ncu DRAM bytes (read + write) of one step launch, per config/format/kernel."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(f"{config}:{fmt}:{kernel}")
    return None if v is None else float(v)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def build_workload(config, fmt):
    from paper_1308_5467_b200 import SparseSymmetricMatrix, workloads as W

    cfg = W.CONFIGS[config]
    op = W.build_matrix(config)
    iv = W.gershgorin_interval(op)
    if fmt in ("csr", "csr-raw") and not isinstance(op, SparseSymmetricMatrix):
        op = SparseSymmetricMatrix(csr=op.csr)
    if fmt == "csr-raw":
        os.environ["SDB_AUTO_STENCIL"] = "0"
    return cfg, op, iv


def kernel_label(dm, n_vec, mode):
    """Name of the step kernel the library runs (sdb_cheb_kernel)."""
    from paper_1308_5467_b200 import _native

    name = _native.load().sdb_cheb_kernel(dm.handle, n_vec, mode).decode()
    detail = {"cheb_step_zmarch": "TMA z-march, ghost-padded planes, register-rolled z terms",
              "cheb_step2_zmarch": "TMA z-march, two fused steps per launch (temporal blocking)",
              "cheb_step_tile": "2.5-D cp.async shared-memory tiles",
              "cheb_step_grid": "row panels", "cheb_step_csr": "CSR row groups",
              "cheb_step_stencil": "generic stencil",
              "cheb_resident": "cluster-resident: all steps in one launch, rows in distributed shared memory",
              "cheb_step_band": "probe-sliced symmetric band (DIA, shared-memory window) + SELL-4 far gathers "
                                "from an L2-resident probe slice"}.get(name, "")
    return f"{name} ({detail})" if detail else name


def nnz_of(op):
    return int(op.csr.nnz) if hasattr(op, "csr") and not hasattr(op, "offsets") else int(op.nnz)


# ---------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port; the reference itself is Python and
# does not travel to the GPU box)


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.lower().startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class CpuSampler:
    """The C restatement of the reference recurrence (oracle/c) on the host
    cores: one probe per pthread (the reference's map_probes thread pool,
    stochastic.py:64-74), ``probes`` probes at a sample degree chosen once from
    a short calibration run so one sample takes about ``target_s`` seconds.
    The recurrence's per-step cost is constant, so the rate nnz*probes*M/t of a
    truncated run is the full run's rate (truncated, extrapolated
    linearly in steps x probes)."""

    def __init__(self, op, iv, cfg, product, probes, target_s):
        from oracle import specdens_oracle as O

        self.op, self.iv, self.cfg, self.product = op, iv, cfg, product
        self.threads = cpu_threads()
        self.probes = probes or min(cfg.n_vec, max(2, self.threads))
        self.pr = np.array([O.draw_probe(cfg.probe_kind, 0, op.dim, l) for l in range(self.probes)])
        cal_deg = min(cfg.degree, 8)
        t = self._run(cal_deg)
        if cal_deg < cfg.degree:
            t = min(t, self._run(cal_deg))
        per_moment = t / cal_deg
        deg = int(target_s / max(per_moment, 1e-9))
        self.degree = max(cal_deg, min(cfg.degree, deg - deg % 2))
        self.truncated = self.degree < cfg.degree

    def _run(self, degree):
        from oracle import c_oracle as C

        t0 = time.perf_counter()
        C.cheb_moments(self.op.csr, self.iv.center, self.iv.halfwidth, degree, self.pr,
                       "doubling" if self.product else "direct", self.threads)
        return time.perf_counter() - t0

    def sample(self):
        return self._run(self.degree)

    def rate(self, secs):
        return nnz_of(self.op) * self.probes * self.degree / secs / 1e9

    def describe(self, secs=None):
        cfg = self.cfg
        cores = min(self.threads, self.probes)
        text = (f"{cfg.name}: {self.probes} of {cfg.n_vec} probes x M={self.degree} of {cfg.degree} moments "
                f"({'doubling' if self.product else 'direct'} recurrence) of the CSR matrix on {cores} host threads "
                f"({cpu_model()}), C restatement of the reference (oracle/c, csr_matvec order, one probe per "
                "pthread)")
        if self.truncated or self.probes < cfg.n_vec:
            text += "; rate of the truncated run = extrapolated full-config rate (time ~ steps x probes)"
        if secs is not None:
            text += f"; {secs:.2f} s wall per sample"
        return text


def cpu_baseline(op, iv, cfg, product, probes=0, target_s=12.0):
    sm = CpuSampler(op, iv, cfg, product, probes, target_s)
    secs = sm.sample()
    value = sm.rate(secs)
    full_s = nnz_of(op) * cfg.n_vec * cfg.degree / value / 1e9
    return {"value": value, "unit": "GNNZ-vec/s", "cores": min(sm.threads, sm.probes), "kind": "port",
            "cpu_model": cpu_model(), "extrapolated": bool(sm.truncated or sm.probes < cfg.n_vec),
            "full_config_seconds_extrapolated": full_s, "sample": sm.describe(secs)}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.config == "C5":
        print(json.dumps({"impl": "reference", "unavailable":
                          "C5's 453M-nnz CSR is not materialised on the host; use tools/config_bench.py --cpu"}),
              flush=True)
        return
    cfg, op, iv = build_workload(args.config, "csr")
    product = not args.direct
    sm = CpuSampler(op, iv, cfg, product, args.cpu_sample_probes, args.cpu_sample_seconds or 4.0)
    times = []
    for i in range(args.warmup + args.steps):
        s = sm.sample()
        if i >= args.warmup:
            times.append(s)
    t = statistics.mean(times)
    value = sm.rate(t)
    cores = min(sm.threads, sm.probes)
    line = {
        "impl": "reference", "metric": "Chebyshev moment steps: nnz*n_vec*deg/s (GNNZ-vec/s)", "value": value,
        "unit": "GNNZ-vec/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, paper_1308_5467_b200/workloads.py)",
        "config": config_dict(cfg, "csr", product, op, 1),
        "cpu_baseline": {"value": value, "unit": "GNNZ-vec/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "extrapolated": bool(sm.truncated or sm.probes < cfg.n_vec),
                         "full_config_seconds_extrapolated": nnz_of(op) * cfg.n_vec * cfg.degree / value / 1e9,
                         "sample": "each step: " + sm.describe(t)},
        "e2e": {"value": value, "unit": "GNNZ-vec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, fmt, product, op, n_gpus):
    return {"workload": f"{cfg.name}: {cfg.description}", "n": int(op.dim), "nnz": nnz_of(op), "degree": cfg.degree,
            "global_probes": cfg.n_vec, "probes_per_gpu": -(-cfg.n_vec // n_gpus), "probe_kind": cfg.probe_kind,
            "grid_points": cfg.grid_points, "damping": "jackson", "format": fmt,
            "moments": "product-formula doubling" if product else "direct",
            "parallelism": f"probe-shard x{n_gpus} (strong: {cfg.n_vec} probes split over the GPUs)",
            "l2": "flushed between timed steps (256 MB write)", "interval": "Gershgorin"}


# ---------------------------------------------------------------------------


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    import paper_1308_5467_b200 as sdb
    from paper_1308_5467_b200 import _native, distributed
    from paper_1308_5467_b200 import engine as E

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    product = not args.direct
    if args.config == "C5" and args.format == "csr":
        args.format = "stencil"  # C5 is generated as the stencil operator (a 453M-nnz CSR is not built)
    cfg, op, iv = build_workload(args.config, args.format)
    if cfg.method != "kpm-jackson":
        raise SystemExit(f"bench.py measures the KPM configs (C1, C2, C3, C5); {cfg.name} is timed by "
                         "tools/config_bench.py")
    n = op.dim
    nnz = nnz_of(op)
    n_vec = cfg.n_vec  # the config's global probe count (strong scaling)
    if n_vec < world:
        raise SystemExit(f"{cfg.name} has {n_vec} probes, fewer than {world} ranks")
    grid = sdb.unit_grid(cfg.grid_points)
    src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=n)
    rowpart = args.config == "C5" and world > 1 and args.format == "stencil"
    first, count = (0, n_vec) if rowpart else distributed.shard_range(n_vec, world, rank)
    # device-resident probes of this rank (drawn once, outside any timing)
    if not rowpart:
        host = src.draw_block(first, count)
        probes_dev = host.to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    mode = _native.SDB_CHEB_DOUBLING if product else _native.SDB_CHEB_DIRECT
    steps_per_probe = (cfg.degree + 1) // 2 if product else cfg.degree
    mapped = sdb.apply_spectral_map(op, iv)
    t_dev = E.to_device(grid, dev)

    if rowpart:
        from paper_1308_5467_b200 import rowpart as RP

        slabs, plan, ros = RP.prepare_rowpartition(op, iv, cfg.degree, src, n_vec, mode, device=local)

    class _Run:
        pass

    def one_step_rowpart():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        zeta_pp = RP.run_rowpartition(slabs, plan, iv.center, iv.halfwidth, cfg.degree, mode, None, ros)
        e1.record()
        zeta, flag = E.mean_moments(zeta_pp, dev)
        E.kpm_density_device(zeta, cfg.degree, n, _native.SDB_DAMP_JACKSON, t_dev, iv.halfwidth, dev)
        torch.cuda.synchronize()
        r = _Run()
        r.step_ms = e0.elapsed_time(e1)
        r.dm = slabs[0].dm
        return r

    def one_step():
        if rowpart:
            return one_step_rowpart()
        run = E.run_chebyshev(mapped, cfg.degree, None, count, mode, device=local, probes=probes_dev,
                              time_steps=True)
        zeta_pp = run.zeta_pp
        if world > 1:
            zeta_pp = distributed.gather_probe_rows(zeta_pp, n_vec)
        zeta, flag = E.mean_moments(zeta_pp, dev)
        E.kpm_density_device(zeta, cfg.degree, n, _native.SDB_DAMP_JACKSON, t_dev, iv.halfwidth, dev)
        return run

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times, kernel_ms = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run = one_step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            kernel_ms.append(run.step_ms)
    if world > 1:
        dist.barrier()
    t_ms = statistics.mean(times)
    k_ms = statistics.mean(kernel_ms)
    if world > 1:
        tt = torch.tensor([t_ms, k_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms, k_ms = float(tt[0]), float(tt[1])
    units = nnz * n_vec * cfg.degree  # the whole job: every rank's probes (or rows)
    value = units / (t_ms * 1e-3) / 1e9

    # ---- e2e through the public API (host probes -> device -> host results) ----
    # cold: a fresh matrix object and a fresh probe source -- the first call
    # uploads the matrix, builds its device layout and draws the probes
    cold_ms = None
    if not rowpart and not args.no_cold:
        cold_op = sdb.SparseSymmetricMatrix(csr=op.csr) if hasattr(op, "csr") and not hasattr(op, "offsets") else \
            sdb.StencilOperator(op.shape, op.offsets, op.weights, op.diag)
        cold_src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=n)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            sdb.estimate_dos(cold_op, iv, "kpm-jackson", cfg.degree, cold_src, n_vec, grid_points=cfg.grid_points,
                             product_formula=product)
        else:
            distributed.estimate_dos_sharded(cold_op, iv, "kpm-jackson", cfg.degree, cold_src, n_vec,
                                             grid_points=cfg.grid_points, product_formula=product)
        torch.cuda.synchronize()
        cold_ms = (time.perf_counter() - t0) * 1e3
        del cold_op, cold_src
    e2e_src = sdb.ProbeVectorSource(cfg.probe_kind, seed=0, dim=n)
    if rowpart:
        def e2e_call():
            return RP.estimate_dos_rowpartition(op, iv, "kpm-jackson", cfg.degree, e2e_src, n_vec,
                                                grid_points=cfg.grid_points, product_formula=product, device=local)
    elif world == 1:
        def e2e_call():
            return sdb.estimate_dos(op, iv, "kpm-jackson", cfg.degree, e2e_src, n_vec, grid_points=cfg.grid_points,
                                    product_formula=product)
    else:
        def e2e_call():
            return distributed.estimate_dos_sharded(op, iv, "kpm-jackson", cfg.degree, e2e_src, n_vec,
                                                    grid_points=cfg.grid_points, product_formula=product)
    for _ in range(max(1, min(args.warmup, 2))):
        e2e_call()
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_call()
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(e2e_t)
    if world > 1:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt[0])
    e2e_value = units / e2e_s / 1e9
    # this rank's probes (Rademacher: packed sign bits, 1/64 of the fp64 bytes) + the unit grid
    h2d = (count * ((n + 7) // 8) if cfg.probe_kind == "rademacher" else 8 * n * count) + 8 * cfg.grid_points
    d2h = 8 * (cfg.degree + 1 + 2 * cfg.grid_points + 1)

    # ---- roofline of the dominant kernel (the fused recurrence step) ----
    dm = run.dm
    ldv = E.block_ldv(count)
    klabel = kernel_label(dm, count, mode)
    kname = klabel.split(" ")[0]
    one_step_bytes = dm.bytes_per_pass + 24 * n * count + (8 * n * count if not product else 0)
    if kname == "cheb_step2_zmarch":
        # fused pairs: per launch the diagonal once, w_k and w_{k-1} read,
        # w_{k+1} and w_{k+2} written; an odd step count ends with one step
        pairs, singles = steps_per_probe // 2, steps_per_probe % 2
        bytes_launch = dm.bytes_per_pass + 32 * n * count
        launches = pairs + singles
        total_bytes = pairs * bytes_launch + singles * one_step_bytes
    elif kname == "cheb_resident":
        # cluster-resident path: every recurrence step of the estimate in ONE launch
        launches = 1
        bytes_launch = steps_per_probe * one_step_bytes
        total_bytes = bytes_launch
    else:
        bytes_launch = one_step_bytes
        launches = steps_per_probe
        total_bytes = launches * one_step_bytes
    avg_launch_s = k_ms * 1e-3 / launches
    achieved = total_bytes / (k_ms * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    traffic = load_traffic(args.config, args.format, kname)
    internal = ("stencil (detected from CSR)" if dm.detected_stencil else
                ("stencil" if dm.format == _native.SDB_FMT_STENCIL else
                 (f"csr split into a symmetric band (half-width {dm.band_half_width}, upper diagonals) + SELL-4 far "
                  "slots" if kname == "cheb_step_band" else "csr")))
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic,
            "kernel": klabel, "peak_source": f"{peak_kind} hbm_gbs",
            "bytes_per_launch": bytes_launch,
            "bytes_model": "algorithmic: M_A + 24*n*n_vec, M_A = 12*nnz + 4*(n+1) for CSR input, 8*n for a stencil "
                           "(SURVEY 8d); not the bytes of the internal layout",
            "launches_per_step": launches,
            "avg_launch_us": avg_launch_s * 1e6, "kernel_share_of_step": k_ms / t_ms, "ldv": ldv}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and nnz <= 100_000_000:
        try:
            cpu = cpu_baseline(op, iv, cfg, product, args.cpu_sample_probes, args.cpu_sample_seconds or 12.0)
        except Exception as exc:  # the baseline must not sink the GPU line
            cpu = {"value": None, "unit": "GNNZ-vec/s", "cores": 1, "kind": "port", "sample": f"failed: {exc}"}

    # my kernels per step: pack + recurrence steps + 2-stage reduce + mean + coefficients + series
    # (+1 layout copy of the probes on the z-march / band paths)
    extra = {"cheb_step_zmarch": 1, "cheb_step2_zmarch": 2, "cheb_step_band": 1}.get(kname, 0)
    gpu_launches = args.steps * (1 + launches + 2 + 1 + 1 + 1 + extra)
    config = config_dict(cfg, args.format, product, op, world)
    config["internal_format"] = internal
    if rowpart:
        config["parallelism"] = f"row-partition x{world} (z-slabs, NCCL halo planes; strong)"
        config["probes_per_gpu"] = n_vec
    line = {
        "metric": "Chebyshev moment steps: nnz*n_vec*deg/s (GNNZ-vec/s)",
        "value": value, "unit": "GNNZ-vec/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, paper_1308_5467_b200/workloads.py)",
        "config": config,
        "roofline": roof, "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "GNNZ-vec/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3, "cache": "warm",
                "cold_first_call_ms": cold_ms,
                "path": "estimate_dos(kpm-jackson) public API; probes from pinned host memory each step "
                        "(Rademacher probes as packed sign bits, expanded to +-1.0 on the device). WARM: the "
                        "matrix handle (uploaded once, cached per host object) and the drawn probe block (cached "
                        "in pinned memory per source) are reused across steps; cold_first_call_ms is one call "
                        "with a fresh matrix object and a fresh probe source (upload + device layout build + "
                        "Philox draws + the estimate)"},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
        "step_rate": {"executed_spmm_gnnz_vec_s": nnz * n_vec * steps_per_probe / (t_ms * 1e-3) / 1e9},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Probe sharding across GPUs (one process per GPU, torch.distributed/NCCL).

Probe recurrences are independent: rank r runs the contiguous
probe range ``shard_range(n_vec, world, r)`` on its own copy of the matrix,
with no data-path collective.  The only exchange is one all-gather of the
per-probe results at the end (moments: n_vec x (M+1) fp64 <= 1 MB; Lanczos:
Ritz values/weights), after which every rank averages in probe order -- so
the result is the same on every rank and independent of the GPU count.

``gather_probe_rows`` works on CPU tensors too (gloo), which is how the N>1
logic is tested without several GPUs.
"""

import numpy as np

from . import _native
from . import engine as E
from .density import DEFAULT_GRID_POINTS, SpectralDensityEstimate, interval_grid, unit_grid
from .errors import NumericalFailure
from .operators import MatvecCounter, apply_spectral_map, as_operator

# every estimate_dos method: Chebyshev / Legendre families gather per-probe
# moment rows, the Lanczos family gathers per-probe Ritz or tridiagonal rows
SHARDED_METHODS = ("kpm", "kpm-jackson", "spectroscopic", "delta-cheb", "kpml", "dgl", "lanczos", "haydock", "cdos")


shard_range = E.shard_range


def gather_probe_rows(rows, n_vec, group=None):
    """All-gather per-probe rows (count_r x k) into the global (n_vec x k) array.

    Ranks may hold different counts (uneven shards); rows are padded to the
    largest shard, gathered with one all_gather_into_tensor, and re-assembled
    in rank order, i.e. probe order.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [shard_range(n_vec, world, r)[1] for r in range(world)]
    cmax = max(counts)
    k = rows.shape[1]
    pad = torch.zeros((cmax, k), dtype=rows.dtype, device=rows.device)
    pad[: rows.shape[0]] = rows
    out = torch.empty((world * cmax, k), dtype=rows.dtype, device=rows.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * cmax: r * cmax + counts[r]] for r in range(world)]
    return torch.cat(parts, dim=0)


def all_gather_probe_moments(zeta_pp, world, group=None):
    """Equal shards (the benchmark's weak-scaling layout)."""
    return gather_probe_rows(zeta_pp, zeta_pp.shape[0] * world, group)


_ShiftedSource = E.ShiftedSource


def estimate_dos_sharded(matrix, interval, method, degree, source, n_vec, sigma=None, grid_points=DEFAULT_GRID_POINTS,
                         product_formula=False, group=None, eta=None):
    """``estimate_dos`` with the probes sharded over the ranks of ``group`` (any method).

    Must be called collectively; every rank returns the same estimate.
    """
    import torch
    import torch.distributed as dist

    from .lanczos import _pool_device, _blur_device, _raise_for_status, lanczos_quadrature_device
    from .operators import resolve

    if method not in SHARDED_METHODS:
        raise ValueError(f"sharded estimates support {SHARDED_METHODS}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    # argument checks come before any work and depend only on the arguments,
    # so every rank raises together (a rank raising alone would leave its
    # peers blocked in the gather)
    if n_vec < world:
        raise ValueError(f"every rank needs at least one probe (n_vec={n_vec}, world size {world})")
    start, count = shard_range(n_vec, world, rank)
    dev = torch.cuda.current_device()
    shifted = _ShiftedSource(source, start)
    counter = MatvecCounter(as_operator(matrix))
    user_counters = resolve(counter).counters[1:] if len(resolve(counter).counters) > 1 else []

    def credit(total):
        # the caller's own MatvecCounter layers see the whole job's MATVECs,
        # as on the single-device paths (E.credit_counters)
        counter.count = int(total)
        for c in user_counters:
            c.count += int(total)
    if product_formula and method not in ("kpm", "kpm-jackson", "spectroscopic", "delta-cheb"):
        raise ValueError("the product formula only applies to Chebyshev moments")
    if method in ("dgl", "lanczos") and (sigma is None or not sigma > 0):
        raise ValueError(f"method {method} requires a positive sigma")
    if method in ("kpm", "kpm-jackson"):
        mode = _native.SDB_CHEB_DOUBLING if product_formula else _native.SDB_CHEB_DIRECT
        run = E.run_chebyshev(apply_spectral_map(counter, interval), degree, shifted, count, mode, device=dev)
        zeta_pp = gather_probe_rows(run.zeta_pp, n_vec, group)
        zeta_dev, flag = E.mean_moments(zeta_pp, dev)
        grid = unit_grid(grid_points)
        damp = _native.SDB_DAMP_JACKSON if method == "kpm-jackson" else _native.SDB_DAMP_NONE
        _, values, density = E.kpm_density_device(zeta_dev, degree, run.n, damp, E.to_device(grid, dev),
                                                  run.resolved.d, dev)
        packed = torch.cat([zeta_dev, values, density, flag.to(torch.float64)]).cpu().numpy()
        m1, g = degree + 1, len(grid)
        if packed[-1] != 0.0 or not np.all(np.isfinite(packed[:m1])):
            raise NumericalFailure(E.SPECTRUM_ESCAPE_HINT)
        credit(n_vec * run.matvecs_per_probe)
        est = SpectralDensityEstimate.from_parts(grid, packed[m1:m1 + g], interval.from_unit(grid),
                                                 packed[m1 + g:m1 + 2 * g], interval,
                                                 method=method, params={"degree": degree, "moments": packed[:m1]})
        if method == "kpm-jackson":
            est.params["damping"] = "jackson"
    elif method in ("spectroscopic", "delta-cheb", "kpml", "dgl"):
        from . import kpm as K
        from .dgl import evaluate_dgl_dos

        legendre = method in ("kpml", "dgl")
        mode = (_native.SDB_LEGENDRE if legendre else
                (_native.SDB_CHEB_DOUBLING if product_formula else _native.SDB_CHEB_DIRECT))
        run = E.run_chebyshev(apply_spectral_map(counter, interval), degree, shifted, count, mode, device=dev)
        zeta_pp = gather_probe_rows(run.zeta_pp, n_vec, group)
        zeta_dev, flag = E.mean_moments(zeta_pp, dev)
        packed = torch.cat([zeta_dev, flag.to(torch.float64)]).cpu().numpy()
        if packed[-1] != 0.0 or not np.all(np.isfinite(packed[:-1])):
            raise NumericalFailure(E.SPECTRUM_ESCAPE_HINT)
        credit(n_vec * run.matvecs_per_probe)
        moments = K.MomentSequence(zeta=packed[:-1], degree=degree, n_vec=n_vec,
                                   basis="legendre" if legendre else "chebyshev", n=run.n)
        grid = unit_grid(grid_points)
        if method == "spectroscopic":
            est = K.spectroscopic_dos(moments, interval, grid, device=dev)
        elif method == "delta-cheb":
            est = K.delta_chebyshev_dos(moments, interval, grid, device=dev)
        elif method == "kpml":
            est = K.evaluate_kpml_dos(moments, interval, grid, device=dev)
        else:
            est = evaluate_dgl_dos(moments, interval, sigma, grid, device=dev)
    elif method == "haydock":
        from .lanczos import lanczos_tridiagonals_device

        grid = interval_grid(interval, grid_points)
        if eta is None:
            eta = interval.width / (2.0 * len(grid))
        if not eta > 0:
            raise ValueError("eta must be positive")
        _, alpha, beta, sd, st = lanczos_tridiagonals_device(counter, degree, shifted, count, device=dev,
                                                             check=False)
        # status rows first: every rank raises the same first error in probe order
        sds = gather_probe_rows(sd.view(-1, 1).to(torch.float64), n_vec, group).view(-1).to(torch.int32)
        sts = gather_probe_rows(st.view(-1, 1).to(torch.float64), n_vec, group).view(-1).to(torch.int32)
        _raise_for_status(sts.cpu().numpy(), sds.cpu().numpy())
        a_all = gather_probe_rows(alpha, n_vec, group).contiguous()
        b_all = gather_probe_rows(beta, n_vec, group).contiguous()
        stream = E.stream_ptr(dev)
        g = E.to_device(grid, dev)
        dens = torch.empty_like(g)
        tpts = torch.empty_like(g)
        trunc = torch.empty(1, dtype=torch.float64, device=dev)
        _native.call("sdb_haydock", E.ptr(a_all), E.ptr(b_all), E.ptr(sds), E.ptr(sts), n_vec, degree, E.ptr(g),
                     g.numel(), float(eta), E.ptr(dens), E.ptr(tpts), E.ptr(trunc), stream)
        packed = torch.cat([dens, trunc]).cpu().numpy()
        credit(sds.sum().item())
        est = SpectralDensityEstimate.from_original(
            grid, packed[:-1], interval, method="haydock",
            params={"M": degree, "n_vec": n_vec, "eta": eta, "truncation_indicator": float(packed[-1])})
    else:
        from .lanczos import DEFAULT_MERGE_RTOL, _cdos_device

        grid = interval_grid(interval, grid_points)
        st_box = []
        _, theta, tau2, sd, _ = lanczos_quadrature_device(counter, degree, shifted, count, device=dev,
                                                          status_out=st_box)
        sds = gather_probe_rows(sd.view(-1, 1).to(torch.float64), n_vec, group).view(-1).to(torch.int32)
        sts = gather_probe_rows(st_box[0].view(-1, 1).to(torch.float64), n_vec, group).view(-1).to(torch.int32)
        _raise_for_status(sts.cpu().numpy(), sds.cpu().numpy())
        th = gather_probe_rows(theta, n_vec, group)
        tw = gather_probe_rows(tau2, n_vec, group)
        stream = E.stream_ptr(dev)
        nodes, weights = _pool_device(th, tw, sds, n_vec, dev, stream)
        credit(sds.sum().item())
        if method == "lanczos":
            dens = _blur_device(nodes, weights, E.to_device(grid, dev), "gaussian", sigma, 1.0, dev, stream)
            density = dens.cpu().numpy()
            est = SpectralDensityEstimate.from_parts(grid, density, grid, density, interval, method="lanczos",
                                                     params={"M": degree, "n_vec": n_vec, "sigma": sigma,
                                                             "ritz_nodes": nodes.cpu().numpy(),
                                                             "ritz_weights": weights.cpu().numpy()})
        else:
            density, mnodes, mweights, cdf = _cdos_device(nodes, weights, interval, grid, DEFAULT_MERGE_RTOL, dev,
                                                          stream)
            est = SpectralDensityEstimate.from_original(
                grid, density, interval, method="cdos",
                params={"cdf": cdf, "nodes": mnodes, "node_weights": mweights, "ritz_nodes": nodes.cpu().numpy(),
                        "ritz_weights": weights.cpu().numpy()})
    est.params.update({"M": degree, "n_vec": n_vec, "matvec_count": counter.count, "world_size": world})
    if product_formula:
        est.params["product_formula"] = True
    return est

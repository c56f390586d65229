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
# methods with a sharded implementation here (one all-gather of per-probe rows)
SHARDED_METHODS = ("kpm", "kpm-jackson", "lanczos")
from .density import DEFAULT_GRID_POINTS, SpectralDensityEstimate, interval_grid, unit_grid
from .errors import NumericalFailure
from .operators import MatvecCounter, apply_spectral_map, as_operator


def shard_range(n_vec, world, rank):
    """Contiguous probe range of ``rank``: sizes differ by at most one."""
    base, extra = divmod(n_vec, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


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


class _ShiftedSource:
    """Probe i of this view is probe start+i of the underlying source."""

    def __init__(self, src, start):
        self.src, self.start, self.dim = src, start, src.dim
        self.kind = getattr(src, "kind", None)
        if hasattr(src, "draw_block_signs"):
            self.draw_block_signs = lambda s, c: src.draw_block_signs(self.start + s, c)

    def draw(self, i):
        return self.src.draw(self.start + i)

    def draw_block(self, start, count):
        from .stochastic import draw_block

        return draw_block(self.src, self.start + start, count)


def estimate_dos_sharded(matrix, interval, method, degree, source, n_vec, sigma=None, grid_points=DEFAULT_GRID_POINTS,
                         product_formula=False, group=None):
    """``estimate_dos`` with the probes sharded over the ranks of ``group``.

    Must be called collectively; every rank returns the same estimate.
    """
    import torch
    import torch.distributed as dist

    from .lanczos import _pool_device, _blur_device, lanczos_quadrature_device

    if method not in SHARDED_METHODS:
        raise ValueError(f"sharded estimates support {SHARDED_METHODS}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    start, count = shard_range(n_vec, world, rank)
    if count < 1:
        raise ValueError("every rank needs at least one probe")
    dev = torch.cuda.current_device()
    shifted = _ShiftedSource(source, start)
    counter = MatvecCounter(as_operator(matrix))
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
        counter.count += n_vec * run.matvecs_per_probe
        est = SpectralDensityEstimate.from_parts(grid, packed[m1:m1 + g], interval.from_unit(grid),
                                                 packed[m1 + g:m1 + 2 * g], interval,
                                                 method=method, params={"degree": degree, "moments": packed[:m1]})
        if method == "kpm-jackson":
            est.params["damping"] = "jackson"
    else:
        if sigma is None or not sigma > 0:
            raise ValueError("method lanczos requires a positive sigma")
        grid = interval_grid(interval, grid_points)
        _, theta, tau2, sd, _ = lanczos_quadrature_device(counter, degree, shifted, count, device=dev)
        th = gather_probe_rows(theta, n_vec, group)
        tw = gather_probe_rows(tau2, n_vec, group)
        sds = gather_probe_rows(sd.view(-1, 1).to(torch.float64), n_vec, group).view(-1).to(torch.int32)
        stream = E.stream_ptr(dev)
        nodes, weights = _pool_device(th, tw, sds, n_vec, dev, stream)
        dens = _blur_device(nodes, weights, E.to_device(grid, dev), "gaussian", sigma, 1.0, dev, stream)
        density = dens.cpu().numpy()
        counter.count = int(sds.sum().item())
        est = SpectralDensityEstimate.from_parts(grid, density, grid, density, interval, method="lanczos",
                                                 params={"M": degree, "n_vec": n_vec, "sigma": sigma,
                                                         "ritz_nodes": nodes.cpu().numpy(),
                                                         "ritz_weights": weights.cpu().numpy()})
    est.params.update({"M": degree, "n_vec": n_vec, "matvec_count": counter.count, "world_size": world})
    if product_formula:
        est.params["product_formula"] = True
    return est

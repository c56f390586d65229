"""Lanczos quadrature on the GPU: drop-in for specdens/lanczos.py (hot path).

  lanczos_factorize      lanczos.py:67-131   -> sdb_lanczos (batch of one)
  prefix_factorization   lanczos.py:134-149  (pure slicing, kept on the host)
  ritz_quadrature        lanczos.py:152-159  -> sdb_ritz_quadrature (first-row QL)
  pool_ritz_quadratures  lanczos.py:170-177  -> sdb_pool_nodes
  blur_nodes             lanczos.py:180-187  -> sdb_blur_nodes
  lanczos_dos            lanczos.py:198-219  -> all probes in lock-step batches,
                                                 quadrature, pooling and blur on device

Haydock / CDOS (lanczos.py:222-368) are outside the hot path.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from . import engine as E
from .density import DEFAULT_GRID_POINTS, RegularizationKernel, SpectralDensityEstimate, interval_grid
from .errors import NumericalFailure
from .operators import device_matrix, resolve

BREAKDOWN_RTOL = 1e-13
REORTH_MODES = ("full", "selective", "none")

# cap on the device memory one batch's Lanczos basis may take
BASIS_BUDGET_BYTES = 64 << 30


@dataclass
class TridiagonalFactorization:
    """alpha (M), beta (M-1), beta_next, optional basis (n x M), breakdown (lanczos.py:33-51)."""

    alpha: np.ndarray
    beta: np.ndarray
    beta_next: float
    basis: np.ndarray = None
    breakdown: bool = False

    @property
    def steps(self):
        return len(self.alpha)


@dataclass
class RitzQuadrature:
    theta: np.ndarray
    tau_sq: np.ndarray
    probe_index: int = None


@dataclass
class LanczosBatch:
    """Device outputs of one lock-step batch."""

    alpha: object        # (count, steps)
    beta: object         # (count, steps)
    steps_done: object   # int32 (count,)
    status: object       # int32 (count,)
    basis: object        # (steps, n, ldv) or None once released
    ldv: int


def _check_args(reorth, steps, dim):
    if reorth not in REORTH_MODES:
        raise ValueError(f"unknown reorth mode {reorth!r}, expected one of {REORTH_MODES}")
    if steps < 1:
        raise ValueError("need at least one Lanczos step")
    if steps > dim:
        raise ValueError(f"steps={steps} exceeds matrix dimension {dim}")


def _run_batch(dm, res, staged, count, steps, reorth, device, stream):
    torch = E._torch()
    lib = _native.load()
    n = res.dim
    basis = torch.empty((steps, n, staged.ldv), dtype=torch.float64, device=device)
    alpha = torch.empty((count, steps), dtype=torch.float64, device=device)
    beta = torch.empty((count, steps), dtype=torch.float64, device=device)
    steps_done = torch.empty(count, dtype=torch.int32, device=device)
    status = torch.empty(count, dtype=torch.int32, device=device)
    need = ctypes.c_size_t()
    _native.check(lib.sdb_lanczos_workspace_size(dm.handle, count, steps, ctypes.byref(need)))
    ws = E.Workspace.get(device, need.value)
    _native.check(lib.sdb_lanczos(dm.handle, res.c, res.d, count, steps, _native.SDB_REORTH[reorth],
                                  E.ptr(staged.block), E.ptr(basis), E.ptr(alpha), E.ptr(beta), E.ptr(steps_done),
                                  E.ptr(status), E.ptr(ws), ws.numel(), stream))
    return LanczosBatch(alpha=alpha, beta=beta, steps_done=steps_done, status=status, basis=basis, ldv=staged.ldv)


def _raise_for_status(status, steps_done, first_index=0):
    """Reproduce the reference's first error in probe order."""
    bad = np.nonzero((status == _native.SDB_LZ_ZERO_START) | (status == _native.SDB_LZ_NONFINITE))[0]
    if bad.size == 0:
        return
    l = int(bad[0])
    if status[l] == _native.SDB_LZ_ZERO_START:
        raise ValueError("starting vector must be nonzero")
    raise NumericalFailure(f"non-finite Lanczos recurrence at step {int(steps_done[l])}")


def _upload_everywhere(base, devices):
    """One matrix upload per distinct device, before any shard thread starts."""
    torch = E._torch()
    for d in sorted(set(int(x) for x in devices)):
        with torch.cuda.device(d):
            device_matrix(base, d, E.stream_ptr(d))
            torch.cuda.current_stream(d).synchronize()


def _batch_size(n, steps, n_vec):
    per_col = 8 * steps * n
    cap = max(1, BASIS_BUDGET_BYTES // max(per_col, 1))
    return int(max(1, min(_native.SDB_MAX_BATCH, n_vec, cap)))


def lanczos_factorize(op, v0, steps, reorth="full", device=None):
    """``steps`` Lanczos iterations from v0 (lanczos.py:67-131), on the GPU."""
    if reorth not in REORTH_MODES:
        raise ValueError(f"unknown reorth mode {reorth!r}, expected one of {REORTH_MODES}")
    if steps < 1:
        raise ValueError("need at least one Lanczos step")
    if steps > op.dim:
        raise ValueError(f"steps={steps} exceeds matrix dimension {op.dim}")
    v0 = np.asarray(v0, dtype=float)
    if np.linalg.norm(v0) == 0.0:
        raise ValueError("starting vector must be nonzero")
    torch = E._torch()
    device = E.require_cuda(device)
    res = resolve(op)
    n = res.dim
    if v0.shape != (n,):
        raise ValueError(f"starting vector has shape {v0.shape}, expected ({n},)")
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        dm = device_matrix(res.base, device, stream)
        probes = E.to_device(v0.reshape(1, n), device)
        staged = E.pack_device_probes(probes, device, stream)
        out = _run_batch(dm, res, staged, 1, steps, reorth, device, stream)
        status = out.status.cpu().numpy()
        sd = out.steps_done.cpu().numpy()
        _raise_for_status(status, sd)
        m = int(sd[0])
        alpha = out.alpha[0, :m].cpu().numpy()
        beta_all = out.beta[0].cpu().numpy()
        basis = out.basis[:m, :, 0].transpose(0, 1).contiguous().cpu().numpy() if m else None
    for c in res.counters:
        c.count += m
    if status[0] == _native.SDB_LZ_BREAKDOWN:
        return TridiagonalFactorization(alpha=alpha, beta=beta_all[: m - 1].copy(), beta_next=0.0, basis=basis,
                                        breakdown=True)
    return TridiagonalFactorization(alpha=alpha, beta=beta_all[: steps - 1].copy(), beta_next=float(beta_all[steps - 1]),
                                    basis=basis)


def prefix_factorization(fact, steps):
    """The factorization the first ``steps`` iterations would give (lanczos.py:134-149)."""
    m = min(steps, fact.steps)
    if m == fact.steps:
        return fact
    return TridiagonalFactorization(
        alpha=fact.alpha[:m].copy(),
        beta=fact.beta[: m - 1].copy(),
        beta_next=float(fact.beta[m - 1]),
        basis=None if fact.basis is None else fact.basis[:, :m],
    )


def _ritz_device(alpha, beta, steps_done, m, device, stream):
    torch = E._torch()
    count = steps_done.numel()
    theta = torch.empty((count, m), dtype=torch.float64, device=device)
    tau2 = torch.empty((count, m), dtype=torch.float64, device=device)
    _native.call("sdb_ritz_quadrature", E.ptr(alpha), E.ptr(beta), E.ptr(steps_done), count, m, E.ptr(theta),
                 E.ptr(tau2), stream)
    return theta, tau2


def ritz_quadrature(fact, probe_index=None, device=None):
    """Ritz values and squared first eigenvector components (lanczos.py:152-159)."""
    torch = E._torch()
    device = E.require_cuda(device)
    m = int(fact.steps)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        a = E.to_device(np.asarray(fact.alpha, dtype=float).reshape(1, m), device)
        b = np.zeros((1, m))
        b[0, : m - 1] = np.asarray(fact.beta, dtype=float)[: m - 1]
        bd = E.to_device(b, device)
        sd = torch.tensor([m], dtype=torch.int32, device=device)
        theta, tau2 = _ritz_device(a, bd, sd, m, device, stream)
        return RitzQuadrature(theta=theta[0].cpu().numpy(), tau_sq=tau2[0].cpu().numpy(), probe_index=probe_index)


def ritz_residual_bounds(fact, device=None):
    """Ritz values with their residual bounds beta_next * |last component| (lanczos.py:162-167)."""
    torch = E._torch()
    device = E.require_cuda(device)
    m = int(fact.steps)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        a = E.to_device(np.asarray(fact.alpha, dtype=float).reshape(1, m), device)
        b = np.zeros((1, m))
        b[0, : m - 1] = np.asarray(fact.beta, dtype=float)[: m - 1]
        b[0, m - 1] = float(fact.beta_next)
        bd = E.to_device(b, device)
        sd = torch.tensor([m], dtype=torch.int32, device=device)
        theta = torch.empty((1, m), dtype=torch.float64, device=device)
        resid = torch.empty((1, m), dtype=torch.float64, device=device)
        _native.call("sdb_ritz_residual_bounds", E.ptr(a), E.ptr(bd), E.ptr(sd), 1, m, E.ptr(theta), E.ptr(resid),
                     stream)
        return theta[0].cpu().numpy(), resid[0].cpu().numpy()


def _pool_device(theta, tau2, steps_done, divisor, device, stream):
    torch = E._torch()
    rows, m = theta.shape
    nodes = torch.empty(rows * m, dtype=torch.float64, device=device)
    weights = torch.empty(rows * m, dtype=torch.float64, device=device)
    count = ctypes.c_int64()
    _native.call("sdb_pool_nodes", E.ptr(theta), E.ptr(tau2), E.ptr(steps_done), rows, m, float(divisor),
                 E.ptr(nodes), E.ptr(weights), ctypes.byref(count), stream)
    return nodes[: count.value], weights[: count.value]


def pool_ritz_quadratures(quads, device=None):
    """Union of per-probe nodes, weights averaged over probes (lanczos.py:170-177)."""
    if not quads:
        raise ValueError("no quadratures to pool")
    torch = E._torch()
    device = E.require_cuda(device)
    m = max(len(q.theta) for q in quads)
    m = max(m, 1)
    th = np.zeros((len(quads), m))
    tw = np.zeros((len(quads), m))
    sd = np.zeros(len(quads), dtype=np.int32)
    for i, q in enumerate(quads):
        k = len(q.theta)
        th[i, :k] = q.theta
        tw[i, :k] = q.tau_sq
        sd[i] = k
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        nodes, weights = _pool_device(E.to_device(th, device), E.to_device(tw, device),
                                      torch.as_tensor(sd).to(device), len(quads), device, stream)
        return RitzQuadrature(theta=nodes.cpu().numpy(), tau_sq=weights.cpu().numpy())


_KERNEL_CODE = {"gaussian": 0, "lorentzian": 1}


def _blur_device(nodes, weights, grid_dev, kind, width, scale, device, stream):
    torch = E._torch()
    out = torch.empty_like(grid_dev)
    _native.call("sdb_blur_nodes", E.ptr(nodes) if nodes.numel() else None,
                 E.ptr(weights) if weights.numel() else None, nodes.numel(), float(scale), _KERNEL_CODE[kind],
                 float(width), E.ptr(grid_dev), grid_dev.numel(), E.ptr(out), stream)
    return out


def blur_nodes(theta, weights, grid, kernel, block=512, device=None):
    """Sum of weighted kernel bumps (lanczos.py:180-187); ``block`` is ignored."""
    torch = E._torch()
    device = E.require_cuda(device)
    grid = np.asarray(grid, dtype=float)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        out = _blur_device(E.to_device(np.asarray(theta, float).ravel(), device),
                           E.to_device(np.asarray(weights, float).ravel(), device),
                           E.to_device(grid.ravel(), device), kernel.kind, kernel.width, 1.0, device, stream)
        return out.cpu().numpy().reshape(grid.shape)


def lanczos_quadrature_device(op, steps, source, n_vec, reorth="full", device=None, probes=None, status_out=None):
    """All probes' (theta, tau2, steps_done) on device, batched in lock-step.

    Returns (res, theta (n_vec, steps), tau2, steps_done, h2d_bytes).
    Raises like the reference on zero starting vectors / non-finite runs;
    with ``status_out`` (a list) the per-probe status tensor is appended
    instead and the caller raises (the sharded path gathers it first, so
    every rank raises the same error).
    """
    torch = E._torch()
    if E.is_device_list(device):  # probe shards, one per list entry; rows gathered on the first device
        primary = E.require_cuda(device)
        res = resolve(op)
        _check_args(reorth, steps, res.dim)
        _upload_everywhere(res.base, device)

        def shard(src, pr, count, d):
            box = []
            out = lanczos_quadrature_device(op, steps, src, count, reorth=reorth, device=d, probes=pr,
                                            status_out=box)
            return out, box[0]

        parts = E.run_sharded(shard, n_vec, device, source=source if probes is None else None, probes=probes)
        with torch.cuda.device(primary):
            theta = torch.cat([p[0][1].to(primary) for p in parts], dim=0)
            tau2 = torch.cat([p[0][2].to(primary) for p in parts], dim=0)
            sd_all = torch.cat([p[0][3].to(primary) for p in parts], dim=0)
            st_all = torch.cat([p[1].to(primary) for p in parts], dim=0)
            h2d = sum(p[0][4] for p in parts)
            if status_out is not None:
                status_out.append(st_all)
                return res, theta, tau2, sd_all, h2d
            _raise_for_status(st_all.cpu().numpy(), sd_all.cpu().numpy())
        return res, theta, tau2, sd_all, h2d
    device = E.require_cuda(device)
    res = resolve(op)
    n = res.dim
    _check_args(reorth, steps, n)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        dm = device_matrix(res.base, device, stream)
        theta = torch.empty((n_vec, steps), dtype=torch.float64, device=device)
        tau2 = torch.empty((n_vec, steps), dtype=torch.float64, device=device)
        sd_all = torch.empty(n_vec, dtype=torch.int32, device=device)
        st_all = torch.empty(n_vec, dtype=torch.int32, device=device)
        h2d = 0
        for start, count in E.batches(n_vec, _batch_size(n, steps, n_vec)):
            if probes is not None:
                staged = E.pack_device_probes(probes[start:start + count], device, stream)
            else:
                staged = E.stage_probes(source, start, count, n, device, stream)
            h2d += staged.h2d_bytes
            out = _run_batch(dm, res, staged, count, steps, reorth, device, stream)
            out.basis = None  # free the basis before the next batch
            th, tw = _ritz_device(out.alpha, out.beta, out.steps_done, steps, device, stream)
            theta[start:start + count] = th
            tau2[start:start + count] = tw
            sd_all[start:start + count] = out.steps_done
            st_all[start:start + count] = out.status
        if status_out is not None:
            status_out.append(st_all)
            return res, theta, tau2, sd_all, h2d
        status = st_all.cpu().numpy()
        sd = sd_all.cpu().numpy()
    _raise_for_status(status, sd)
    return res, theta, tau2, sd_all, h2d


def lanczos_dos(op, interval, steps, source, n_vec, sigma, grid=None, threads=None, reorth="full", device=None):
    """Gaussian-blurred average of per-probe Ritz quadratures (lanczos.py:198-219)."""
    if not sigma > 0:
        raise ValueError("sigma must be positive")
    if grid is None:
        grid = interval_grid(interval, DEFAULT_GRID_POINTS)
    grid = np.asarray(grid, dtype=float)
    torch = E._torch()
    devices, device = device, E.require_cuda(device)
    res, theta, tau2, sd, _ = lanczos_quadrature_device(op, steps, source, n_vec, reorth=reorth, device=devices)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        nodes, weights = _pool_device(theta, tau2, sd, n_vec, device, stream)
        dens = _blur_device(nodes, weights, E.to_device(grid, device), "gaussian", sigma, 1.0, device, stream)
        density = dens.cpu().numpy()
        nodes_h = nodes.cpu().numpy()
        weights_h = weights.cpu().numpy()
    for c in res.counters:
        c.count += int(sd.sum().item())
    return SpectralDensityEstimate.from_parts(
        grid, density, grid, density, interval, method="lanczos",
        params={"M": steps, "n_vec": n_vec, "sigma": sigma, "ritz_nodes": nodes_h, "ritz_weights": weights_h},
    )


# ---------------------------------------------------------------------------
# Haydock resolvent (lanczos.py:222-293): the batched
# Lanczos tridiagonals stay on the device and one kernel evaluates every
# probe's continued fraction and truncation diagnostic per grid point.


def lanczos_tridiagonals_device(op, steps, source, n_vec, reorth="full", device=None, probes=None, check=True):
    """All probes' (alpha, beta, steps_done, status) on device (sdb_lanczos layout).

    ``check=False`` leaves raising on the status row to the caller."""
    torch = E._torch()
    if E.is_device_list(device):
        primary = E.require_cuda(device)
        res = resolve(op)
        _check_args(reorth, steps, res.dim)
        _upload_everywhere(res.base, device)
        parts = E.run_sharded(lambda src, pr, count, d: lanczos_tridiagonals_device(
            op, steps, src, count, reorth=reorth, device=d, probes=pr, check=False), n_vec, device,
            source=source if probes is None else None, probes=probes)
        with torch.cuda.device(primary):
            alpha, beta, sd_all, st_all = (torch.cat([p[k].to(primary) for p in parts], dim=0) for k in (1, 2, 3, 4))
            if check:
                _raise_for_status(st_all.cpu().numpy(), sd_all.cpu().numpy())
        return res, alpha, beta, sd_all, st_all
    device = E.require_cuda(device)
    res = resolve(op)
    n = res.dim
    _check_args(reorth, steps, n)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        dm = device_matrix(res.base, device, stream)
        alpha = torch.empty((n_vec, steps), dtype=torch.float64, device=device)
        beta = torch.empty((n_vec, steps), dtype=torch.float64, device=device)
        sd_all = torch.empty(n_vec, dtype=torch.int32, device=device)
        st_all = torch.empty(n_vec, dtype=torch.int32, device=device)
        for start, count in E.batches(n_vec, _batch_size(n, steps, n_vec)):
            if probes is not None:
                staged = E.pack_device_probes(probes[start:start + count], device, stream)
            else:
                staged = E.stage_probes(source, start, count, n, device, stream)
            out = _run_batch(dm, res, staged, count, steps, reorth, device, stream)
            out.basis = None
            alpha[start:start + count] = out.alpha
            beta[start:start + count] = out.beta
            sd_all[start:start + count] = out.steps_done
            st_all[start:start + count] = out.status
        if not check:
            return res, alpha, beta, sd_all, st_all
        status = st_all.cpu().numpy()
        sd = sd_all.cpu().numpy()
    _raise_for_status(status, sd)
    return res, alpha, beta, sd_all, st_all


def _resolvent(alpha, beta, z, want_cf, want_w, device=None):
    torch = E._torch()
    device = E.require_cuda(device)
    alpha = np.asarray(alpha, dtype=float)
    beta = np.asarray(beta, dtype=float)
    z = np.asarray(z, dtype=complex)
    m = len(alpha)
    zf = np.ascontiguousarray(z.ravel())
    nz = zf.size
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        a = E.to_device(alpha, device)
        b = E.to_device(beta if m > 1 else np.zeros(1), device)
        zd = E.to_device(zf.view(np.float64), device)
        cf = torch.empty(2 * nz, dtype=torch.float64, device=device) if want_cf else None
        w0 = torch.empty(2 * nz, dtype=torch.float64, device=device) if want_w else None
        wl = torch.empty(2 * nz, dtype=torch.float64, device=device) if want_w else None
        scratch = torch.empty(max(4 * m * nz, 1), dtype=torch.float64, device=device) if want_w else None
        _native.call("sdb_tridiag_resolvent", E.ptr(a), E.ptr(b), m, E.ptr(zd), nz, E.ptr(cf), E.ptr(w0), E.ptr(wl),
                     E.ptr(scratch), stream)

        def host(t):
            return None if t is None else t.cpu().numpy().view(np.complex128).reshape(z.shape)

        return host(cf), host(w0), host(wl)


def continued_fraction_resolvent(alpha, beta, z, device=None):
    """Bottom-up continued fraction for e1^T (zI - T)^{-1} e1, vectorized in z (lanczos.py:222-227)."""
    return _resolvent(alpha, beta, z, True, False, device)[0]


def tridiagonal_resolvent_first(alpha, beta, z, device=None):
    """(w_0, w_{M-1}) of (zI - T) w = e1 by the Thomas algorithm (lanczos.py:230-260)."""
    _, w0, wl = _resolvent(alpha, beta, z, False, True, device)
    return w0, wl


def haydock_dos(op, interval, steps, source, n_vec, eta=None, grid=None, threads=None, reorth="full", device=None):
    """Lorentzian-regularized DOS from the (1,1) resolvent continued fraction (lanczos.py:263-293).

    ``eta`` defaults to half a grid spacing; params["truncation_indicator"] is
    max beta_next |w_{M-1}| over probes and grid points.
    """
    if grid is None:
        grid = interval_grid(interval, DEFAULT_GRID_POINTS)
    grid = np.asarray(grid, dtype=float)
    if eta is None:
        eta = interval.width / (2.0 * len(grid))
    if not eta > 0:
        raise ValueError("eta must be positive")
    torch = E._torch()
    devices, device = device, E.require_cuda(device)
    res, alpha, beta, sd, st = lanczos_tridiagonals_device(op, steps, source, n_vec, reorth=reorth, device=devices)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        g = E.to_device(grid, device)
        dens = torch.empty_like(g)
        tpts = torch.empty_like(g)
        trunc = torch.empty(1, dtype=torch.float64, device=device)
        _native.call("sdb_haydock", E.ptr(alpha), E.ptr(beta), E.ptr(sd), E.ptr(st), n_vec, steps, E.ptr(g),
                     g.numel(), float(eta), E.ptr(dens), E.ptr(tpts), E.ptr(trunc), stream)
        packed = torch.cat([dens, trunc]).cpu().numpy()
    for c in res.counters:
        c.count += int(sd.sum().item())
    density = packed[:-1]
    return SpectralDensityEstimate.from_original(
        grid, density, interval, method="haydock",
        params={"M": steps, "n_vec": n_vec, "eta": eta, "truncation_indicator": float(packed[-1])},
    )


# ---------------------------------------------------------------------------
# CDOS (lanczos.py:296-368): a monotone PCHIP spline through the pooled
# cumulative staircase, averaged over each grid cell -- one merge pass, the
# PCHIP slopes and the cell averages on the device (sdb_cdos_refine).

DEFAULT_MERGE_RTOL = 1e-10


class PchipCdf:
    """The CDF spline of a CDOS estimate: breakpoints, values and PCHIP slopes
    (what SciPy's PchipInterpolator holds).  Calling it evaluates the cubic
    Hermite pieces on the host -- an inspection helper, not the estimator."""

    def __init__(self, x, y, d):
        self.x, self.y, self.d = np.asarray(x), np.asarray(y), np.asarray(d)

    def __call__(self, xq):
        xq = np.asarray(xq, dtype=float)
        i = np.clip(np.searchsorted(self.x, xq, side="right") - 1, 0, len(self.x) - 2)
        h = self.x[i + 1] - self.x[i]
        s = xq - self.x[i]
        m = (self.y[i + 1] - self.y[i]) / h
        t = (self.d[i] + self.d[i + 1] - 2 * m) / h
        return self.y[i] + self.d[i] * s + ((m - self.d[i]) / h - t) * s**2 + t / h * s**3


def _cdos_device(theta_dev, weights_dev, interval, grid, merge_rtol, device, stream):
    torch = E._torch()
    count = theta_dev.numel()
    nodes = torch.empty(max(count, 1), dtype=torch.float64, device=device)
    wts = torch.empty_like(nodes)
    sx = torch.empty(count + 2, dtype=torch.float64, device=device)
    sy = torch.empty_like(sx)
    sd = torch.empty_like(sx)
    g = E.to_device(grid, device)
    dens = torch.empty_like(g)
    k = ctypes.c_int64(0)
    _native.call("sdb_cdos_refine", E.ptr(theta_dev) if count else None, E.ptr(weights_dev) if count else None,
                 count, float(merge_rtol * interval.width), float(interval.lambda_lb), float(interval.lambda_ub),
                 E.ptr(g), g.numel(), E.ptr(dens), E.ptr(nodes), E.ptr(wts), E.ptr(sx), E.ptr(sy), E.ptr(sd),
                 ctypes.byref(k), stream)
    kk = k.value
    packed = torch.cat([dens, nodes[:kk], wts[:kk], sx[:kk + 2], sy[:kk + 2], sd[:kk + 2]]).cpu().numpy()
    n = g.numel()
    parts = np.split(packed, np.cumsum([n, kk, kk, kk + 2, kk + 2]))
    return parts[0], parts[1], parts[2], PchipCdf(parts[3], parts[4], parts[5])


def cdos_refine(quad, interval, grid=None, merge_rtol=DEFAULT_MERGE_RTOL, device=None):
    """Differentiate a monotone spline through the cumulative staircase (lanczos.py:296-349)."""
    if grid is None:
        grid = interval_grid(interval, DEFAULT_GRID_POINTS)
    grid = np.asarray(grid, dtype=float)
    torch = E._torch()
    device = E.require_cuda(device)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        th = E.to_device(np.asarray(quad.theta, dtype=float).ravel(), device)
        tw = E.to_device(np.asarray(quad.tau_sq, dtype=float).ravel(), device)
        order = torch.argsort(th, stable=True)
        density, nodes, weights, cdf = _cdos_device(th[order].contiguous(), tw[order].contiguous(), interval, grid,
                                                    merge_rtol, device, stream)
    return SpectralDensityEstimate.from_original(
        grid, density, interval, method="cdos", params={"cdf": cdf, "nodes": nodes, "node_weights": weights},
    )


def cdos_dos(op, interval, steps, source, n_vec, grid=None, threads=None, reorth="full", device=None):
    """Pool per-probe Ritz quadratures and refine the cumulative staircase (lanczos.py:352-368)."""
    _check_args(reorth, steps, resolve(op).dim)
    if grid is None:
        grid = interval_grid(interval, DEFAULT_GRID_POINTS)
    grid = np.asarray(grid, dtype=float)
    torch = E._torch()
    devices, device = device, E.require_cuda(device)
    res, theta, tau2, sd, _ = lanczos_quadrature_device(op, steps, source, n_vec, reorth=reorth, device=devices)
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        nodes_p, weights_p = _pool_device(theta, tau2, sd, n_vec, device, stream)  # sorted by theta
        density, nodes, weights, cdf = _cdos_device(nodes_p, weights_p, interval, grid, DEFAULT_MERGE_RTOL, device,
                                                    stream)
        ritz_nodes = nodes_p.cpu().numpy()
        ritz_weights = weights_p.cpu().numpy()
    for c in res.counters:
        c.count += int(sd.sum().item())
    est = SpectralDensityEstimate.from_original(
        grid, density, interval, method="cdos", params={"cdf": cdf, "nodes": nodes, "node_weights": weights},
    )
    est.params.update({"M": steps, "n_vec": n_vec, "ritz_nodes": ritz_nodes, "ritz_weights": ritz_weights})
    return est

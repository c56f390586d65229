"""Front door: ``estimate_dos`` for the GPU methods (specdens/compare.py:74-141).

Methods on the hot path: ``kpm``, ``kpm-jackson`` (direct or product-formula
moments) and ``lanczos``.  For the KPM methods the whole chain -- moments,
probe mean, finiteness check, coefficients, Clenshaw, 1/sqrt(1-t^2) and the
1/d unmapping -- stays on the device and the host reads back the moments and
the density once.  The moment-sharing variants ``spectroscopic``,
``delta-cheb`` (same Chebyshev moments) and ``kpml`` (Legendre moments from
the same fused kernels) run through the same kernels.  ``dgl``
runs its gamma recurrence on the same Legendre moments, and ``haydock``
evaluates the batched Lanczos tridiagonals' resolvents on the device
(§8(f)-3); ``cdos`` refines the pooled Ritz staircase with a monotone
spline on the device (sdb_cdos_refine).
"""

import time

import numpy as np

from . import _native
from . import engine as E
from . import kpm as K
from .density import DEFAULT_GRID_POINTS, SpectralDensityEstimate, interval_grid, unit_grid
from .errors import NumericalFailure
from .dgl import evaluate_dgl_dos
from .lanczos import cdos_dos, haydock_dos, lanczos_dos
from .operators import MatvecCounter, apply_spectral_map, as_operator

CHEBYSHEV_METHODS = ("kpm", "kpm-jackson", "spectroscopic", "delta-cheb")
LEGENDRE_METHODS = ("kpml", "dgl")
LANCZOS_METHODS = ("lanczos", "haydock", "cdos")
ALL_METHODS = CHEBYSHEV_METHODS + LEGENDRE_METHODS + LANCZOS_METHODS
GPU_METHODS = ALL_METHODS


def analytic_matvec_count(method, degree, n_vec, product_formula=False):
    """degree MATVECs per probe, (degree+1)//2 with the product formula (compare.py:74-79)."""
    if method == "exact":
        return 0
    per_probe = (degree + 1) // 2 if product_formula else degree
    return n_vec * per_probe


def kpm_dos_device(mapped, degree, source, n_vec, damping, grid, product_formula, device=None, probes=None,
                   time_steps=False):
    """Moments -> DOS entirely on device.  Returns (zeta, values, density, run)."""
    torch = E._torch()
    mode = _native.SDB_CHEB_DOUBLING if product_formula else _native.SDB_CHEB_DIRECT
    # the grid goes up first: its (synchronous, pageable) copy would otherwise make the host wait for
    # the moment run before it can queue the evaluation kernels behind it
    primary = E.require_cuda(device)
    with torch.cuda.device(primary):
        t_dev = E.to_device(grid, primary)
    run = E.run_chebyshev(mapped, degree, source, n_vec, mode, device=device, probes=probes, time_steps=time_steps)
    dev = run.zeta_pp.device
    with torch.cuda.device(dev):
        zeta_dev, flag = E.mean_moments(run.zeta_pp, dev)
        damp = _native.SDB_DAMP_JACKSON if damping == "jackson" else _native.SDB_DAMP_NONE
        _, values, density = E.kpm_density_device(zeta_dev, degree, run.n, damp, t_dev, run.resolved.d, dev)
        packed = torch.cat([zeta_dev, values, density, flag.to(torch.float64)]).cpu().numpy()
    m1, g = degree + 1, len(grid)
    zeta = packed[:m1]
    vals = packed[m1:m1 + g]
    dens = packed[m1 + g:m1 + 2 * g]
    nonfinite = packed[-1] != 0.0
    return zeta, vals, dens, nonfinite, run


def estimate_dos(matrix, interval, method, degree, source, n_vec, sigma=None, eta=None,
                 grid_points=DEFAULT_GRID_POINTS, threads=None, product_formula=False, device=None, devices=None):
    """Run one estimator on the GPU; params carry the MATVEC count (compare.py:82-141).

    ``devices=[0, 1, ...]`` shards the probes over several GPUs of this
    process (one contiguous probe range, host thread and stream per entry;
    the matrix is replicated); the per-probe moment / Ritz / tridiagonal rows
    are gathered on ``devices[0]`` in probe order and evaluated there, so the
    call keeps the reference's single-process signature.  Per-probe results
    do not depend on the sharding beyond the rounding of their dot-product
    reduction trees (<= 1e-13 relative).
    """
    if devices is not None:
        if device is not None:
            raise ValueError("pass either device or devices")
        device = [int(d) for d in devices]
        if not device:
            raise ValueError("devices must name at least one CUDA device")
    if method not in ALL_METHODS:
        raise ValueError(f"unknown method {method!r}, expected one of {ALL_METHODS}")
    if product_formula and method not in CHEBYSHEV_METHODS:
        raise ValueError("the product formula only applies to Chebyshev moments")
    if method in ("dgl", "lanczos") and (sigma is None or not sigma > 0):
        raise ValueError(f"method {method} requires a positive sigma")
    if method not in GPU_METHODS:
        raise NotImplementedError(
            f"method {method!r} is outside the accelerated hot path; GPU methods are {GPU_METHODS}"
        )

    counter = MatvecCounter(as_operator(matrix))
    start = time.perf_counter()
    if method in ("kpm", "kpm-jackson"):
        if n_vec < 1:
            raise ValueError("need at least one probe vector")
        if degree < 0:
            raise ValueError("degree must be non-negative")
        mapped = apply_spectral_map(counter, interval)
        grid = unit_grid(grid_points)
        damping = "jackson" if method == "kpm-jackson" else "none"
        zeta, values, density, nonfinite, run = kpm_dos_device(mapped, degree, source, n_vec, damping, grid,
                                                               product_formula, device=device)
        E.credit_counters(run.resolved, n_vec, run.matvecs_per_probe)
        if nonfinite or not np.all(np.isfinite(zeta)):
            raise NumericalFailure(E.SPECTRUM_ESCAPE_HINT)
        est = SpectralDensityEstimate.from_parts(grid, values, interval.from_unit(grid), density, interval,
                                                 method="kpm", params={"degree": degree})
        if method == "kpm-jackson":
            est.method = "kpm-jackson"
            est.params["damping"] = "jackson"
        est.params["moments"] = zeta
    elif method in ("spectroscopic", "delta-cheb"):
        mapped = apply_spectral_map(counter, interval)
        compute = K.moments_via_product_formula if product_formula else K.compute_chebyshev_moments
        moments = compute(mapped, degree, source, n_vec, threads, device=device)
        grid = unit_grid(grid_points)
        if method == "spectroscopic":
            est = K.spectroscopic_dos(moments, interval, grid, device=device)
        else:
            est = K.delta_chebyshev_dos(moments, interval, grid, device=device)
    elif method in LEGENDRE_METHODS:
        mapped = apply_spectral_map(counter, interval)
        moments = K.compute_legendre_moments(mapped, degree, source, n_vec, threads, device=device)
        if method == "kpml":
            est = K.evaluate_kpml_dos(moments, interval, unit_grid(grid_points), device=device)
        else:
            est = evaluate_dgl_dos(moments, interval, sigma, unit_grid(grid_points), device=device)
    else:
        grid = interval_grid(interval, grid_points)
        if method == "lanczos":
            est = lanczos_dos(counter, interval, degree, source, n_vec, sigma, grid, threads, device=device)
        elif method == "haydock":
            est = haydock_dos(counter, interval, degree, source, n_vec, eta, grid, threads, device=device)
        else:
            est = cdos_dos(counter, interval, degree, source, n_vec, grid, threads, device=device)
    est.params.update({
        "M": degree,
        "n_vec": n_vec,
        "matvec_count": counter.count,
        "wall_time_s": time.perf_counter() - start,
    })
    if devices is not None:
        est.params["devices"] = list(device)
    if sigma is not None:
        est.params.setdefault("sigma", sigma)
    if product_formula:
        est.params["product_formula"] = True
    return est


# ---------------------------------------------------------------------------
# Repeated method x degree sweep (compare.py:144-284), SURVEY §8(f)-4.
#
# The device does the sweep's work in three batched passes instead of
# reps x n_vec independent runs: the probes of every repetition (stream = rep)
# are drawn on the host exactly as the reference draws them and stacked into
# one device block, then ONE Chebyshev, ONE Legendre and ONE batched Lanczos
# run cover all reps x n_vec recurrences at the largest degree; each rep's
# moments are its probe-ordered mean of that run, every smaller degree is an
# exact prefix (kpm.py:49-59, lanczos.py:134-149).  Per degree, the Ritz
# quadratures of all probes come from one QL launch, pooled and blurred per
# rep; Haydock evaluates each rep's prefix tridiagonals in one launch.  The
# scoring references (the blurred exact spectrum on the two grids and at the
# sup-Gaussian centres) are computed once, and the per-estimate errors stay on
# the device until one read at the end.

from dataclasses import dataclass, field  # noqa: E402

from .density import RegularizationKernel  # noqa: E402
from .kpm import MomentSequence  # noqa: E402
from .lanczos import (  # noqa: E402
    DEFAULT_MERGE_RTOL,
    _blur_device,
    _cdos_device,
    _pool_device,
    _ritz_device,
    lanczos_tridiagonals_device,
)
from .metrics import DEFAULT_SUP_CENTERS, check_sup_gaussian_grid, sup_gaussian_device  # noqa: E402
from .operators import estimate_spectral_interval, resolve  # noqa: E402
from .reference import blurred_spectrum_device, dense_eigensolve  # noqa: E402
from .stochastic import ProbeVectorSource, draw_block  # noqa: E402

# scored with the sup-Gaussian metric (their output approximates the raw spike
# density); the rest are compared pointwise to the matching blur (compare.py:67-69)
SPIKE_ESTIMATORS = ("kpm", "kpm-jackson", "spectroscopic", "delta-cheb", "kpml", "cdos")


@dataclass
class MethodComparisonRow:
    """Aggregated accuracy of one method at one degree across repetitions (compare.py:144-154)."""

    method: str
    degree: int
    matvec_count: int
    error_mean: float
    error_std: float
    mass_mean: float
    errors: np.ndarray = field(repr=False, default=None)


def _stacked_probes(kind, seed, dim, reps, n_vec, device):
    """(reps*n_vec, dim) device block: rep r's probes are ProbeVectorSource(kind, seed, dim, stream=r)."""
    torch = E._torch()
    out = torch.empty((reps * n_vec, dim), dtype=torch.float64, device=device)
    for rep in range(reps):
        blk = draw_block(ProbeVectorSource(kind, seed, dim, stream=rep), 0, n_vec)
        out[rep * n_vec:(rep + 1) * n_vec].copy_(torch.as_tensor(np.asarray(blk, dtype=np.float64)))
    return out


def _rep_moments(mapped, m_max, probes, reps, n_vec, mode, basis, device):
    """One moment run over every rep's probes; each rep's probe-ordered mean as a MomentSequence."""
    torch = E._torch()
    run = E.run_chebyshev(mapped, m_max, None, reps * n_vec, mode, device=device, probes=probes)
    means, flags = [], []
    for rep in range(reps):
        z, f = E.mean_moments(run.zeta_pp[rep * n_vec:(rep + 1) * n_vec], device)
        means.append(z)
        flags.append(f)
    zeta = torch.stack(means).cpu().numpy()
    if int(torch.cat(flags).max().item()) != 0 or not np.all(np.isfinite(zeta)):
        raise NumericalFailure(E.SPECTRUM_ESCAPE_HINT)
    return [MomentSequence(zeta=zeta[rep], degree=m_max, n_vec=n_vec, basis=basis, n=run.n) for rep in range(reps)]


def run_method_comparison(matrix, methods, degrees, sigma, eta=None, n_vec=100, reps=10, seed=0,
                          probe_kind="gaussian", grid_points=512, threads=None, interval=None, spectrum=None,
                          device=None):
    """Repeat a method x degree sweep and aggregate errors and masses (compare.py:162-284).

    Same arguments, validation order, common random numbers (probe stream =
    repetition), exact-prefix slicing, scoring protocol and rows as the
    reference; ``threads`` is ignored.
    """
    for m in methods:
        if m not in ALL_METHODS and m != "exact":
            raise ValueError(f"unknown method {m!r}, expected one of {ALL_METHODS}")
    if not sigma > 0:
        raise ValueError("sigma must be positive")
    degrees = sorted(set(int(m) for m in degrees))
    if not degrees or degrees[0] < 1:
        raise ValueError("degrees must be positive")
    torch = E._torch()
    device = E.require_cuda(device)
    op = as_operator(matrix)
    if interval is None:
        interval = estimate_spectral_interval(op, seed=seed, device=device)
    if spectrum is None:
        spectrum = dense_eigensolve(op, device=device)
    if eta is None:
        eta = sigma

    m_max = degrees[-1]
    unit_pts = unit_grid(grid_points)
    lam_grid = interval_grid(interval, grid_points)
    unit_lam = interval.from_unit(unit_pts)  # lambda_grid of the unit-grid estimates
    gauss = RegularizationKernel("gaussian", sigma)

    need_cheb = any(m in CHEBYSHEV_METHODS for m in methods)
    need_leg = any(m in LEGENDRE_METHODS for m in methods)
    need_lan = any(m in LANCZOS_METHODS for m in methods)
    if any(m in SPIKE_ESTIMATORS and m != "cdos" for m in methods):
        check_sup_gaussian_grid(unit_lam, sigma)
    if "cdos" in methods:
        check_sup_gaussian_grid(lam_grid, sigma)

    errors = {(m, deg): [] for m in methods for deg in degrees}
    masses = {(m, deg): [] for m in methods for deg in degrees}
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        n = resolve(op).dim
        probes = _stacked_probes(probe_kind, seed, n, reps, n_vec, device)
        mapped = apply_spectral_map(op, interval)
        cheb = (_rep_moments(mapped, m_max, probes, reps, n_vec, _native.SDB_CHEB_DIRECT, "chebyshev", device)
                if need_cheb else None)
        leg = (_rep_moments(mapped, m_max, probes, reps, n_vec, _native.SDB_LEGENDRE, "legendre", device)
               if need_leg else None)
        if need_lan:
            steps = min(m_max, n)
            _, alpha, beta, sd, st = lanczos_tridiagonals_device(op, steps, None, reps * n_vec, device=device,
                                                                 probes=probes)

        # scoring references, computed once
        eig_dev = E.to_device(spectrum.eigenvalues, device)
        lam_dev = E.to_device(lam_grid, device)
        unit_lam_dev = E.to_device(unit_lam, device)
        centers_dev = E.to_device(np.linspace(interval.lambda_lb, interval.lambda_ub, DEFAULT_SUP_CENTERS), device)
        exact_centers = blurred_spectrum_device(spectrum, gauss, centers_dev, device, eig_dev)
        exact_lam = blurred_spectrum_device(spectrum, gauss, lam_dev, device, eig_dev)
        exact_unit = (blurred_spectrum_device(spectrum, gauss, unit_lam_dev, device, eig_dev)
                      if "dgl" in methods else None)
        exact_lam_h = exact_lam.cpu().numpy()

        def score_spike(density_dev, grid_dev):
            return sup_gaussian_device(exact_centers, grid_dev, density_dev, centers_dev, sigma, device)

        def score_blur(density_dev, ref_dev):
            return torch.max(torch.abs(density_dev - ref_dev))

        for rep in range(reps):
            sl = slice(rep * n_vec, (rep + 1) * n_vec)
            for deg in degrees:
                if need_lan:
                    dp = min(deg, steps)
                    a_p = alpha[:, :dp].contiguous()
                    b_p = beta[:, :dp].contiguous()
                    sd_p = torch.clamp(sd, max=dp).to(torch.int32)
                    if "lanczos" in methods or "cdos" in methods:
                        th, tw = _ritz_device(a_p[sl], b_p[sl], sd_p[sl], dp, device, stream)
                        nodes, weights = _pool_device(th, tw, sd_p[sl], n_vec, device, stream)
                    if "lanczos" in methods:
                        lan_dens = _blur_device(nodes, weights, lam_dev, "gaussian", sigma, 1.0, device, stream)
                    if "cdos" in methods:
                        cdos_h = _cdos_device(nodes, weights, interval, lam_grid, DEFAULT_MERGE_RTOL, device, stream)[0]
                    if "haydock" in methods:
                        hay_dens = torch.empty_like(lam_dev)
                        _native.call("sdb_haydock", E.ptr(a_p[sl]), E.ptr(b_p[sl]), E.ptr(sd_p[sl]), E.ptr(st[sl]),
                                     n_vec, dp, E.ptr(lam_dev), lam_dev.numel(), float(eta), E.ptr(hay_dens), None,
                                     None, stream)
                for method in methods:
                    if method == "exact":
                        # oracle scored against itself: a zero-error control row
                        err = score_blur(exact_lam, exact_lam)
                        mass = float(np.trapezoid(exact_lam_h, lam_grid))
                    elif method in CHEBYSHEV_METHODS or method in LEGENDRE_METHODS:
                        moments = (cheb if method in CHEBYSHEV_METHODS else leg)[rep].truncated(deg)
                        if method == "kpm":
                            est = K.evaluate_kpm_dos(K.moments_to_coefficients(moments, "none", device=device),
                                                     interval, unit_pts, device=device)
                        elif method == "kpm-jackson":
                            est = K.evaluate_kpm_dos(K.moments_to_coefficients(moments, "jackson", device=device),
                                                     interval, unit_pts, device=device)
                        elif method == "spectroscopic":
                            est = K.spectroscopic_dos(moments, interval, unit_pts, device=device)
                        elif method == "delta-cheb":
                            est = K.delta_chebyshev_dos(moments, interval, unit_pts, device=device)
                        elif method == "kpml":
                            est = K.evaluate_kpml_dos(moments, interval, unit_pts, device=device)
                        else:
                            est = evaluate_dgl_dos(moments, interval, sigma, unit_pts, device=device)
                        if method in SPIKE_ESTIMATORS:
                            err = score_spike(E.to_device(est.density, device), unit_lam_dev)
                        else:
                            err = score_blur(E.to_device(est.density, device), exact_unit)
                        mass = est.mass()
                    elif method == "cdos":
                        err = score_spike(E.to_device(cdos_h, device), lam_dev)
                        mass = float(np.trapezoid(cdos_h, lam_grid))
                    else:
                        dens = lan_dens if method == "lanczos" else hay_dens
                        err = score_blur(dens, exact_lam)
                        mass = float(np.trapezoid(dens.cpu().numpy(), lam_grid))
                    errors[(method, deg)].append(err)
                    masses[(method, deg)].append(mass)
        keys = list(errors)
        flat = torch.stack([e for k in keys for e in errors[k]]).cpu().numpy() if keys else np.zeros(0)

    rows = []
    pos = 0
    per_key = {}
    for k in keys:
        per_key[k] = flat[pos:pos + len(errors[k])]
        pos += len(errors[k])
    for method in methods:
        for deg in degrees:
            errs = np.asarray(per_key[(method, deg)], dtype=float)
            rows.append(MethodComparisonRow(
                method=method,
                degree=deg,
                matvec_count=analytic_matvec_count(method, deg, n_vec),
                error_mean=float(errs.mean()),
                error_std=float(errs.std(ddof=1)) if reps > 1 else 0.0,
                mass_mean=float(np.mean(masses[(method, deg)])),
                errors=errs,
            ))
    return rows


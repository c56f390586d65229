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
(§8(f)-3).  The remaining reference method (cdos, a monotone-spline
refinement of the Lanczos staircase) is outside the accelerated path and
raises ``NotImplementedError``.
"""

import time

import numpy as np

from . import _native
from . import engine as E
from . import kpm as K
from .density import DEFAULT_GRID_POINTS, SpectralDensityEstimate, interval_grid, unit_grid
from .errors import NumericalFailure
from .dgl import evaluate_dgl_dos
from .lanczos import haydock_dos, lanczos_dos
from .operators import MatvecCounter, apply_spectral_map, as_operator

CHEBYSHEV_METHODS = ("kpm", "kpm-jackson", "spectroscopic", "delta-cheb")
LEGENDRE_METHODS = ("kpml", "dgl")
LANCZOS_METHODS = ("lanczos", "haydock", "cdos")
ALL_METHODS = CHEBYSHEV_METHODS + LEGENDRE_METHODS + LANCZOS_METHODS
GPU_METHODS = ("kpm", "kpm-jackson", "spectroscopic", "delta-cheb", "kpml", "dgl", "lanczos", "haydock")


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
    run = E.run_chebyshev(mapped, degree, source, n_vec, mode, device=device, probes=probes, time_steps=time_steps)
    dev = run.zeta_pp.device
    with torch.cuda.device(dev):
        zeta_dev, flag = E.mean_moments(run.zeta_pp, dev)
        t_dev = E.to_device(grid, dev)
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
                 grid_points=DEFAULT_GRID_POINTS, threads=None, product_formula=False, device=None):
    """Run one estimator on the GPU; params carry the MATVEC count (compare.py:82-141)."""
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
        else:
            est = haydock_dos(counter, interval, degree, source, n_vec, eta, grid, threads, device=device)
    est.params.update({
        "M": degree,
        "n_vec": n_vec,
        "matvec_count": counter.count,
        "wall_time_s": time.perf_counter() - start,
    })
    if sigma is not None:
        est.params.setdefault("sigma", sigma)
    if product_formula:
        est.params["product_formula"] = True
    return est

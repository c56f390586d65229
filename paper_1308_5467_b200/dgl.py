"""Delta-Gauss-Legendre estimator on the GPU: drop-in for specdens/dgl.py.

The Legendre moments come from the fused step kernels (kpm.compute_legendre_
moments); the gamma_k recurrence (one expansion centre per thread, halted at
its stability cutoff) and the weighted sum over k run in ``sdb_dgl``.

  gamma_zero                dgl.py:35-39    (closed form, host helper)
  compute_dgl_coefficients  dgl.py:92-106   -> sdb_dgl (gamma / psi tables)
  evaluate_dgl_dos          dgl.py:109-132  -> sdb_dgl (weighted sums, / n sqrt(2 pi) sigma_m)
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from . import engine as E
from .density import SpectralDensityEstimate, unit_grid
from .errors import NumericalFailure

DEFAULT_DGL_TOL = 1e-6


@dataclass(frozen=True)
class DGLCoefficients:
    """Gamma and psi sequences for one expansion center, up to the cutoff (dgl.py:25-32)."""

    gamma: np.ndarray
    psi: np.ndarray
    effective_degree: int
    center: float
    sigma: float


def gamma_zero(t, sigma):
    """gamma_0(t): the Gaussian bump's mass over [-1, 1] (dgl.py:35-39)."""
    from scipy.special import erf

    t = np.asarray(t, dtype=float)
    s = np.sqrt(2.0) * sigma
    return sigma * np.sqrt(np.pi / 2.0) * (erf((1.0 - t) / s) + erf((1.0 + t) / s))


def _check(sigma, tol, max_degree):
    if not sigma > 0:
        raise ValueError("sigma must be positive")
    if not tol > 0:
        raise ValueError("tol must be positive")
    if max_degree < 0:
        raise ValueError("max degree must be non-negative")


def _run(weights, degree, t, sigma, tol, divisor, want_tables, device):
    torch = E._torch()
    device = E.require_cuda(device)
    t = np.asarray(t, dtype=float)
    n_pts = t.size
    with torch.cuda.device(device):
        stream = E.stream_ptr(device)
        td = E.to_device(t, device)
        wd = None if weights is None else E.to_device(weights, device)
        values = torch.empty(n_pts, dtype=torch.float64, device=device) if weights is not None else None
        gamma = psi = None
        if want_tables:
            gamma = torch.empty((degree + 1, n_pts), dtype=torch.float64, device=device)
            psi = torch.empty((degree + 1, n_pts), dtype=torch.float64, device=device)
        eff = torch.empty(n_pts, dtype=torch.int32, device=device)
        failed = torch.zeros(1, dtype=torch.int32, device=device)
        _native.call("sdb_dgl", E.ptr(wd), int(degree), E.ptr(td), n_pts, float(sigma), float(tol), float(divisor),
                     E.ptr(values), E.ptr(gamma), E.ptr(psi), E.ptr(eff), E.ptr(failed), stream)
        f = int(failed.item())
        if f:
            raise NumericalFailure(f"gamma recurrence lost stability at k={f}")
        host = lambda x: None if x is None else x.cpu().numpy()  # noqa: E731
        return host(values), host(gamma), host(psi), host(eff)


def compute_dgl_coefficients(t, sigma, max_degree, tol=DEFAULT_DGL_TOL, device=None):
    """Gamma coefficients for one center, truncated at the stability cutoff (dgl.py:92-106)."""
    if not -1.0 < t < 1.0:
        raise ValueError("expansion center must lie inside (-1, 1)")
    _check(sigma, tol, max_degree)
    _, gamma, psi, eff = _run(None, max_degree, np.array([t]), sigma, tol, 1.0, True, device)
    k = int(eff[0])
    return DGLCoefficients(gamma=gamma[: k + 1, 0].copy(), psi=psi[: k + 1, 0].copy(), effective_degree=k,
                           center=float(t), sigma=float(sigma))


def evaluate_dgl_dos(moments, interval, sigma, grid=None, tol=DEFAULT_DGL_TOL, device=None):
    """Gaussian-regularized density from Legendre moments (dgl.py:109-132)."""
    if moments.basis != "legendre":
        raise ValueError("DGL evaluation needs legendre moments")
    if not sigma > 0:
        raise ValueError("sigma must be positive")
    t = unit_grid() if grid is None else np.asarray(grid, dtype=float)
    if np.any(np.abs(t) >= 1.0):
        raise ValueError("evaluation points must lie inside (-1, 1)")
    sigma_m = sigma / interval.halfwidth
    _check(sigma_m, tol, moments.degree)
    k = np.arange(moments.degree + 1)
    weighted = (k + 0.5) * moments.zeta
    divisor = moments.n * np.sqrt(2.0 * np.pi) * sigma_m
    values, _, _, eff = _run(weighted, moments.degree, t, sigma_m, tol, divisor, False, device)
    return SpectralDensityEstimate.from_mapped(
        t, values, interval, method="dgl",
        params={"degree": moments.degree, "sigma": sigma, "effective_degree": int(eff.max())},
    )

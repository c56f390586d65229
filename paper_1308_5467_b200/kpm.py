"""Kernel polynomial method on the GPU: drop-in for specdens/kpm.py.

Same names, arguments, return types and error behaviour as the reference
(kpm.py:33-250); the arithmetic runs in the sm_100a kernels of
libspecdens_b200.so:

  compute_chebyshev_moments   kpm.py:143-147  -> K1 direct mode + K2 + mean
  moments_via_product_formula kpm.py:157-198  -> K1 doubling mode + K2 + mean
  jackson_damping             kpm.py:84-93    -> sdb_jackson_damping
  moments_to_coefficients     kpm.py:201-208  -> sdb_kpm_coefficients
  evaluate_chebyshev_series   kpm.py:211-217  -> sdb_chebyshev_series
  evaluate_kpm_dos            kpm.py:244-250  -> sdb_chebyshev_series (+1/sqrt(1-t^2), /d)
  compute_legendre_moments    kpm.py:110-124, :150-154 -> K1 direct-mode kernels, Legendre update
  evaluate_legendre_series    kpm.py:220-231  -> sdb_legendre_series
  evaluate_kpml_dos           kpm.py:298-308  -> sdb_legendre_series (/d)
  spectroscopic_dos           kpm.py:253-266  -> coefficients + series kernels
  delta_chebyshev_dos         kpm.py:269-295  -> series kernel per truncation degree

``threads`` is accepted for signature compatibility and ignored: the probes
already run concurrently on the device and results are deterministic.
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from . import engine as E
from .density import DEFAULT_GRID_POINTS, EDGE_GUARD, SpectralDensityEstimate, unit_grid
from .errors import NumericalFailure

MOMENT_BASES = ("chebyshev", "legendre")
SPECTRUM_ESCAPE_HINT = E.SPECTRUM_ESCAPE_HINT


@dataclass(frozen=True)
class MomentSequence:
    """Averaged raw moments zeta_k, k = 0..degree (kpm.py:33-59)."""

    zeta: np.ndarray
    degree: int
    n_vec: int
    basis: str
    n: int

    def __post_init__(self):
        if self.basis not in MOMENT_BASES:
            raise ValueError(f"unknown moment basis {self.basis!r}")
        if len(self.zeta) != self.degree + 1:
            raise ValueError("moment array length must be degree + 1")

    def truncated(self, degree):
        """Exact prefix (kpm.py:49-59)."""
        if degree > self.degree:
            raise ValueError(f"cannot extend degree {self.degree} to {degree}")
        return MomentSequence(zeta=self.zeta[: degree + 1], degree=degree, n_vec=self.n_vec, basis=self.basis,
                              n=self.n)


@dataclass(frozen=True)
class DampingKernel:
    kind: str = "none"

    def __post_init__(self):
        if self.kind not in ("none", "jackson"):
            raise ValueError(f"unknown damping kind {self.kind!r}")

    def coefficients(self, degree):
        if self.kind == "none":
            return np.ones(degree + 1)
        return jackson_damping(degree)


def _as_damping(damping):
    if isinstance(damping, DampingKernel):
        return damping
    if hasattr(damping, "kind") and not isinstance(damping, str):
        return DampingKernel(kind=damping.kind)
    return DampingKernel(kind=damping)


_DAMP_CODE = {"none": _native.SDB_DAMP_NONE, "jackson": _native.SDB_DAMP_JACKSON}


def _moments(op, degree, source, n_vec, mode, device=None):
    run = E.run_chebyshev(op, degree, source, n_vec, mode, device=device)
    dev = run.zeta_pp.device
    zeta_dev, flag = E.mean_moments(run.zeta_pp, dev)
    zeta = zeta_dev.cpu().numpy()
    E.credit_counters(run.resolved, n_vec, run.matvecs_per_probe)
    if int(flag.item()) != 0 or not np.all(np.isfinite(zeta)):
        raise NumericalFailure(SPECTRUM_ESCAPE_HINT)
    basis = "legendre" if mode == _native.SDB_LEGENDRE else "chebyshev"
    return MomentSequence(zeta=zeta, degree=degree, n_vec=n_vec, basis=basis, n=run.n)


def compute_chebyshev_moments(op, degree, source, n_vec, threads=None, device=None):
    """Chebyshev moments via the three-term recurrence: degree MATVECs/probe."""
    if n_vec < 1:
        raise ValueError("need at least one probe vector")
    if degree < 0:
        raise ValueError("degree must be non-negative")
    return _moments(op, degree, source, n_vec, _native.SDB_CHEB_DIRECT, device)


def compute_legendre_moments(op, degree, source, n_vec, threads=None, device=None):
    """Legendre moments via (k+1)L_{k+1} = (2k+1)tL_k - kL_{k-1} (kpm.py:110-124, :150-154)."""
    if n_vec < 1:
        raise ValueError("need at least one probe vector")
    if degree < 0:
        raise ValueError("degree must be non-negative")
    return _moments(op, degree, source, n_vec, _native.SDB_LEGENDRE, device)


def moments_via_product_formula(op, degree, source, n_vec, threads=None, max_stored_vectors=None, device=None):
    """Chebyshev moments from half the MATVECs (kpm.py:157-198).

    The reference stores v_0..v_p; the fused kernel needs none of that
    history (each step emits zeta_{2k+1} and zeta_{2k+2} from the rows it
    just produced), but the storage-cap contract is kept.
    """
    if degree < 0:
        raise ValueError("degree must be non-negative")
    p = (degree + 1) // 2
    if max_stored_vectors is not None and p + 1 > max_stored_vectors:
        raise ValueError(f"product formula needs {p + 1} stored vectors, cap is {max_stored_vectors}")
    if n_vec < 1:
        raise ValueError("need at least one probe vector")
    return _moments(op, degree, source, n_vec, _native.SDB_CHEB_DOUBLING, device)


def jackson_damping(degree, device=None):
    """Jackson damping factors g_k, k = 0..degree (kpm.py:84-93)."""
    torch = E._torch()
    device = E.require_cuda(device)
    with torch.cuda.device(device):
        g = torch.empty(int(degree) + 1, dtype=torch.float64, device=device)
        _native.call("sdb_jackson_damping", int(degree), E.ptr(g), E.stream_ptr(device))
        return g.cpu().numpy()


def moments_to_coefficients(moments, damping="none", device=None):
    """mu_k = (2 - delta_k0)/(n pi) zeta_k g_k (kpm.py:201-208)."""
    if moments.basis != "chebyshev":
        raise ValueError("expansion coefficients need chebyshev moments")
    kind = _as_damping(damping).kind
    torch = E._torch()
    device = E.require_cuda(device)
    with torch.cuda.device(device):
        z = E.to_device(moments.zeta, device)
        mu = torch.empty_like(z)
        _native.call("sdb_kpm_coefficients", E.ptr(z), int(moments.degree), int(moments.n), _DAMP_CODE[kind],
                     E.ptr(mu), E.stream_ptr(device))
        return mu.cpu().numpy()


def evaluate_chebyshev_series(coeffs, t, device=None):
    """Clenshaw evaluation of sum_k coeffs[k] T_k(t) (kpm.py:211-217)."""
    coeffs = np.asarray(coeffs, dtype=float)
    t_arr = np.asarray(t, dtype=float)
    torch = E._torch()
    device = E.require_cuda(device)
    with torch.cuda.device(device):
        c = E.to_device(coeffs, device)
        tt = E.to_device(t_arr.ravel(), device)
        out = torch.empty_like(tt)
        _native.call("sdb_chebyshev_series", E.ptr(c), len(coeffs) - 1, E.ptr(tt), tt.numel(), 0, 1.0,
                     E.ptr(out), None, E.stream_ptr(device))
        return out.cpu().numpy().reshape(t_arr.shape)


def _checked_unit_points(grid):
    t = unit_grid(DEFAULT_GRID_POINTS) if grid is None else np.asarray(grid, dtype=float)
    if np.any(np.abs(t) > 1.0 - EDGE_GUARD):
        raise ValueError(
            f"evaluation points must satisfy |t| <= 1 - {EDGE_GUARD} "
            "(the Chebyshev weight is singular at the interval edges)"
        )
    return t


def evaluate_kpm_dos(coeffs, interval, grid=None, device=None):
    """KPM density sum_k mu_k T_k(t)/sqrt(1 - t^2) on a unit grid (kpm.py:244-250)."""
    t = _checked_unit_points(grid)
    coeffs = np.asarray(coeffs, dtype=float)
    torch = E._torch()
    device = E.require_cuda(device)
    d = float(interval.halfwidth)
    with torch.cuda.device(device):
        c = E.to_device(coeffs, device)
        tt = E.to_device(t, device)
        values = torch.empty_like(tt)
        density = torch.empty_like(tt)
        _native.call("sdb_chebyshev_series", E.ptr(c), len(coeffs) - 1, E.ptr(tt), tt.numel(), 1, d,
                     E.ptr(values), E.ptr(density), E.stream_ptr(device))
        v = values.cpu().numpy()
        den = density.cpu().numpy()
    return SpectralDensityEstimate.from_parts(
        t, v, interval.from_unit(t), den, interval, method="kpm", params={"degree": len(coeffs) - 1}
    )


def evaluate_legendre_series(coeffs, t, device=None):
    """Forward-recurrence evaluation of sum_k coeffs[k] L_k(t) (kpm.py:220-231)."""
    coeffs = np.asarray(coeffs, dtype=float)
    t_arr = np.asarray(t, dtype=float)
    torch = E._torch()
    device = E.require_cuda(device)
    with torch.cuda.device(device):
        c = E.to_device(coeffs, device)
        tt = E.to_device(t_arr.ravel(), device)
        out = torch.empty_like(tt)
        _native.call("sdb_legendre_series", E.ptr(c), len(coeffs) - 1, E.ptr(tt), tt.numel(), 1.0, E.ptr(out), None,
                     E.stream_ptr(device))
        return out.cpu().numpy().reshape(t_arr.shape)


def evaluate_kpml_dos(moments, interval, grid=None, device=None):
    """Legendre-basis density sum_k (k + 1/2) zeta_k/n L_k(t), no edge weight (kpm.py:298-308)."""
    if moments.basis != "legendre":
        raise ValueError("KPML evaluation needs legendre moments")
    t = _checked_unit_points(grid)
    k = np.arange(moments.degree + 1)
    coeffs = (k + 0.5) * moments.zeta / moments.n
    torch = E._torch()
    device = E.require_cuda(device)
    d = float(interval.halfwidth)
    with torch.cuda.device(device):
        c = E.to_device(coeffs, device)
        tt = E.to_device(t, device)
        values = torch.empty_like(tt)
        density = torch.empty_like(tt)
        _native.call("sdb_legendre_series", E.ptr(c), int(moments.degree), E.ptr(tt), tt.numel(), d, E.ptr(values),
                     E.ptr(density), E.stream_ptr(device))
        v = values.cpu().numpy()
        den = density.cpu().numpy()
    return SpectralDensityEstimate.from_parts(t, v, interval.from_unit(t), den, interval, method="kpml",
                                              params={"degree": moments.degree})


def spectroscopic_dos(moments, interval, grid=None, device=None):
    """Undamped KPM with the top coefficient halved (kpm.py:253-266)."""
    coeffs = moments_to_coefficients(moments, damping="none", device=device)
    if moments.degree >= 1:
        coeffs = coeffs.copy()
        coeffs[-1] *= 0.5
    est = evaluate_kpm_dos(coeffs, interval, grid=grid, device=device)
    est.method = "spectroscopic"
    return est


def delta_chebyshev_dos(moments, interval, grid=None, degrees=None, device=None):
    """Per-point-degree truncations of the undamped Chebyshev expansion (kpm.py:269-295).

    Points sharing a truncation degree go through the same Clenshaw kernel as
    KPM, so the uniform case is bit-identical to undamped KPM.
    """
    t = _checked_unit_points(grid)
    if degrees is None:
        degrees = np.full(len(t), moments.degree, dtype=int)
    degrees = np.asarray(degrees, dtype=int)
    if degrees.shape != t.shape:
        raise ValueError("degrees must match the grid point for point")
    if np.any(degrees < 0) or np.any(degrees > moments.degree):
        raise ValueError(f"per-point degrees must lie in [0, {moments.degree}]")
    coeffs = moments_to_coefficients(moments, damping="none", device=device)
    torch = E._torch()
    device = E.require_cuda(device)
    d = float(interval.halfwidth)
    values = np.empty_like(t)
    density = np.empty_like(t)
    with torch.cuda.device(device):
        c = E.to_device(coeffs, device)
        for deg in np.unique(degrees):
            mask = degrees == deg
            tt = E.to_device(t[mask], device)
            v = torch.empty_like(tt)
            den = torch.empty_like(tt)
            _native.call("sdb_chebyshev_series", E.ptr(c), int(deg), E.ptr(tt), tt.numel(), 1, d, E.ptr(v),
                         E.ptr(den), E.stream_ptr(device))
            values[mask] = v.cpu().numpy()
            density[mask] = den.cpu().numpy()
    return SpectralDensityEstimate.from_parts(t, values, interval.from_unit(t), density, interval,
                                              method="delta-cheb",
                                              params={"degree": moments.degree, "degrees": degrees})

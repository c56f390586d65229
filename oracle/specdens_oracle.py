"""CPU ORACLE — test infrastructure only, never the product path.

A plain NumPy/SciPy restatement of the reference's hot-path algorithms
(/root/reference/pkg/src/specdens, cited per function).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference legs
may import it, and only as the checker or the timed CPU baseline.

Pinning: ``tests/golden/make_golden.py`` runs the reference itself (importable
in the build container) on fixed seeded inputs and stores its outputs under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks this module against
those fixtures (bit-for-bit where the arithmetic order is the same).

Third-party arithmetic the reference delegates to (pinned only as
``numpy>=2.0, scipy>=1.13`` in pkg/pyproject.toml:9-12; this image has NumPy
2.3.5, SciPy 1.18.1):
  * SciPy ``csr_matvec`` (csr @ x): y_i = sum over the row's stored entries in
    storage order -- used here through the same SciPy call;
  * LAPACK ``?stevd`` via ``scipy.linalg.eigh_tridiagonal`` -- same call;
  * NumPy Philox/SeedSequence probe streams -- same calls.
"""

import numpy as np
import scipy.sparse as sp
from scipy.linalg import eigh_tridiagonal

EDGE_GUARD = 1e-6
BREAKDOWN_RTOL = 1e-13


class OracleNumericalFailure(RuntimeError):
    pass


# ---- probes: stochastic.py:40-54 -------------------------------------------------
def draw_probe(kind, seed, dim, index, stream=0):
    if kind == "basis":
        v = np.zeros(dim)
        v[index] = np.sqrt(dim)
        return v
    ss = np.random.SeedSequence(seed, spawn_key=(stream, index))
    rng = np.random.Generator(np.random.Philox(ss))
    if kind == "gaussian":
        return rng.standard_normal(dim)
    return rng.integers(0, 2, dim) * 2.0 - 1.0


def as_csr(matrix):
    if sp.issparse(matrix):
        return sp.csr_array(matrix)
    if hasattr(matrix, "csr"):
        return matrix.csr
    return sp.csr_array(np.asarray(matrix, dtype=float))


# ---- mapped matvec: matrix.py:101-102, :125-126 -------------------------------------
def mapped_matvec(csr, c, d, x):
    return (csr @ x - c * x) / d


# ---- kpm.py:96-107 --------------------------------------------------------------------
def chebyshev_probe_moments(csr, c, d, degree, v0):
    zeta = np.empty(degree + 1)
    zeta[0] = v0 @ v0
    if degree == 0:
        return zeta
    v_prev = v0
    v_cur = mapped_matvec(csr, c, d, v0)
    zeta[1] = v0 @ v_cur
    for k in range(2, degree + 1):
        v_cur, v_prev = 2.0 * mapped_matvec(csr, c, d, v_cur) - v_prev, v_cur
        zeta[k] = v0 @ v_cur
    return zeta


# ---- kpm.py:174-189 (product formula, one probe) ------------------------------------------
def product_formula_probe_moments(csr, c, d, degree, v0):
    p = (degree + 1) // 2
    stored = np.empty((p + 1, len(v0)))
    stored[0] = v0
    if p >= 1:
        stored[1] = mapped_matvec(csr, c, d, stored[0])
    for j in range(2, p + 1):
        stored[j] = 2.0 * mapped_matvec(csr, c, d, stored[j - 1]) - stored[j - 2]
    zeta = np.empty(degree + 1)
    for k in range(0, p + 1):
        if k <= degree:
            zeta[k] = v0 @ stored[k]
    for k in range(p + 1, degree + 1):
        a = (k + 1) // 2
        b = k - a
        zeta[k] = 2.0 * (stored[a] @ stored[b]) - zeta[a - b]
    return zeta


# ---- doubling identities of the north star (the form the GPU kernel computes) ----------------
def doubling_probe_moments(csr, c, d, degree, v0):
    """zeta_{2k} = 2<w_k,w_k> - zeta_0, zeta_{2k+1} = 2<w_{k+1},w_k> - zeta_1 (kpm.py:162-163)."""
    zeta = np.empty(degree + 1)
    zeta[0] = v0 @ v0
    if degree == 0:
        return zeta
    w_prev, w = None, v0
    k = 0
    while True:
        w_next = mapped_matvec(csr, c, d, w) if k == 0 else 2.0 * mapped_matvec(csr, c, d, w) - w_prev
        if 2 * k + 1 <= degree:
            r = w_next @ w
            zeta[2 * k + 1] = r if k == 0 else 2.0 * r - zeta[1]
        if 2 * k + 2 <= degree:
            zeta[2 * k + 2] = 2.0 * (w_next @ w_next) - zeta[0]
        k += 1
        if 2 * k + 1 > degree:
            break
        w_prev, w = w, w_next
    return zeta


# ---- kpm.py:110-124 (Legendre recurrence, one probe) -----------------------------------------
def legendre_probe_moments(csr, c, d, degree, v0):
    zeta = np.empty(degree + 1)
    zeta[0] = v0 @ v0
    if degree == 0:
        return zeta
    v_prev = v0
    v_cur = mapped_matvec(csr, c, d, v0)
    zeta[1] = v0 @ v_cur
    for k in range(1, degree):
        v_cur, v_prev = ((2 * k + 1) * mapped_matvec(csr, c, d, v_cur) - k * v_prev) / (k + 1.0), v_cur
        zeta[k + 1] = v0 @ v_cur
    return zeta


# ---- kpm.py:127-140 ----------------------------------------------------------------------
def average_moments(per_probe):
    zeta = np.mean(np.asarray(per_probe), axis=0)
    if not np.all(np.isfinite(zeta)):
        raise OracleNumericalFailure("non-finite moments")
    return zeta


def chebyshev_moments(matrix, c, d, degree, kind, seed, n_vec, mode="direct", stream=0, indices=None):
    """Per-probe moments (n_vec x (degree+1)) over probe indices 0..n_vec-1."""
    csr = as_csr(matrix)
    n = csr.shape[0]
    fn = {"direct": chebyshev_probe_moments, "product": product_formula_probe_moments,
          "doubling": doubling_probe_moments, "legendre": legendre_probe_moments}[mode]
    idx = range(n_vec) if indices is None else indices
    return np.array([fn(csr, c, d, degree, draw_probe(kind, seed, n, l, stream)) for l in idx])


# ---- kpm.py:84-93, :201-217, :234-250 ------------------------------------------------------
def jackson_damping(degree):
    k = np.arange(degree + 1)
    a = np.pi / (degree + 2)
    return ((1.0 - k / (degree + 2)) * np.sin(a) * np.cos(k * a)
            + np.sin(k * a) * np.cos(a) / (degree + 2)) / np.sin(a)


def moments_to_coefficients(zeta, n, damping="none"):
    degree = len(zeta) - 1
    g = np.ones(degree + 1) if damping == "none" else jackson_damping(degree)
    prefactor = np.full(degree + 1, 2.0 / (n * np.pi))
    prefactor[0] = 1.0 / (n * np.pi)
    return prefactor * zeta * g


def evaluate_chebyshev_series(coeffs, t):
    b1 = np.zeros_like(t)
    b2 = np.zeros_like(t)
    for c in coeffs[:0:-1]:
        b1, b2 = 2.0 * t * b1 - b2 + c, b1
    return t * b1 - b2 + coeffs[0]


def unit_grid(n_pts):
    h = 2.0 / n_pts
    return -1.0 + (np.arange(n_pts) + 0.5) * h


def interval_grid(lb, ub, n_pts, pad=0.0):
    lo, hi = lb - pad, ub + pad
    h = (hi - lo) / n_pts
    return lo + (np.arange(n_pts) + 0.5) * h


def evaluate_kpm_dos(coeffs, d, t):
    """(values, density) on unit points t (kpm.py:244-250, density.py:124-136)."""
    if np.any(np.abs(t) > 1.0 - EDGE_GUARD):
        raise ValueError("grid point too close to the interval edge")
    values = evaluate_chebyshev_series(coeffs, t) / np.sqrt(1.0 - t * t)
    return values, values / d


# ---- kpm.py:220-231, :253-308 (moment-sharing variants) -------------------------------------
def evaluate_legendre_series(coeffs, t):
    acc = coeffs[0] * np.ones_like(t)
    if len(coeffs) == 1:
        return acc
    l_prev = np.ones_like(t)
    l_cur = np.asarray(t, dtype=float)
    acc = acc + coeffs[1] * l_cur
    for k in range(1, len(coeffs) - 1):
        l_cur, l_prev = ((2 * k + 1) * t * l_cur - k * l_prev) / (k + 1.0), l_cur
        acc += coeffs[k + 1] * l_cur
    return acc


def kpml_dos(zeta, n, d, t):
    """(values, density): sum_k (k + 1/2) zeta_k/n L_k(t), unmapped by 1/d (kpm.py:298-308)."""
    k = np.arange(len(zeta))
    values = evaluate_legendre_series((k + 0.5) * zeta / n, t)
    return values, values / d


def spectroscopic_dos(zeta, n, d, t):
    """Undamped KPM with the top coefficient halved (kpm.py:253-266)."""
    coeffs = moments_to_coefficients(zeta, n, "none")
    if len(zeta) >= 2:
        coeffs = coeffs.copy()
        coeffs[-1] *= 0.5
    return evaluate_kpm_dos(coeffs, d, t)


def delta_chebyshev_dos(zeta, n, d, t, degrees):
    """Per-point truncation degrees of the undamped series (kpm.py:269-295)."""
    coeffs = moments_to_coefficients(zeta, n, "none")
    values = np.empty_like(t)
    for deg in np.unique(degrees):
        mask = degrees == deg
        ts = t[mask]
        values[mask] = evaluate_chebyshev_series(coeffs[: deg + 1], ts) / np.sqrt(1.0 - ts * ts)
    return values, values / d


# ---- lanczos.py:67-131 ---------------------------------------------------------------------
def lanczos_factorize(csr, v0, steps, reorth="full", c=0.0, d=1.0):
    """Returns (alpha, beta, beta_next, basis, breakdown)."""
    def matvec(x):
        y = csr @ x
        return y if (c == 0.0 and d == 1.0) else (y - c * x) / d

    v0 = np.asarray(v0, dtype=float)
    nrm = np.linalg.norm(v0)
    if nrm == 0.0:
        raise ValueError("starting vector must be nonzero")
    dim = csr.shape[0]
    basis = np.empty((dim, steps))
    basis[:, 0] = v0 / nrm
    alpha = np.empty(steps)
    beta = np.empty(max(steps - 1, 0))
    sqrt_eps = np.sqrt(np.finfo(float).eps)
    beta_next = 0.0
    tscale = 0.0
    for j in range(steps):
        w = matvec(basis[:, j])
        if j > 0:
            w = w - beta[j - 1] * basis[:, j - 1]
        a = float(basis[:, j] @ w)
        w -= a * basis[:, j]
        alpha[j] = a
        if reorth == "full":
            for _ in range(2):
                w -= basis[:, : j + 1] @ (basis[:, : j + 1].T @ w)
        elif reorth == "selective":
            overlaps = basis[:, : j + 1].T @ w
            big = np.abs(overlaps) > sqrt_eps * np.linalg.norm(w)
            if big.any():
                w -= basis[:, : j + 1][:, big] @ overlaps[big]
        b = float(np.linalg.norm(w))
        if not (np.isfinite(a) and np.isfinite(b)):
            raise OracleNumericalFailure(f"non-finite Lanczos recurrence at step {j + 1}")
        tscale = max(tscale, abs(a), b)
        if j == steps - 1:
            beta_next = b
        elif b <= BREAKDOWN_RTOL * max(tscale, 1.0):
            return alpha[: j + 1], beta[:j], 0.0, basis[:, : j + 1], True
        else:
            beta[j] = b
            basis[:, j + 1] = w / b
    return alpha, beta, beta_next, basis, False


# ---- lanczos.py:152-159, :170-187 ---------------------------------------------------------------
def ritz_quadrature(alpha, beta):
    if len(alpha) == 1:
        return alpha.copy(), np.ones(1)
    theta, y = eigh_tridiagonal(alpha, beta)
    return theta, y[0, :] ** 2


def pool(quads):
    theta = np.concatenate([q[0] for q in quads])
    tau = np.concatenate([q[1] for q in quads]) / len(quads)
    order = np.argsort(theta)
    return theta[order], tau[order]


def gaussian(x, sigma):
    return np.exp(-0.5 * (x / sigma) ** 2) / np.sqrt(2.0 * np.pi * sigma * sigma)


def blur_nodes(theta, weights, grid, sigma, block=512):
    out = np.zeros_like(grid, dtype=float)
    for start in range(0, len(theta), block):
        th = theta[start:start + block]
        wt = weights[start:start + block]
        out += gaussian(grid[None, :] - th[:, None], sigma).T @ wt
    return out


def lanczos_dos(matrix, steps, kind, seed, n_vec, sigma, grid, reorth="full", indices=None):
    """(density, nodes, weights, per-probe (alpha, beta, beta_next))."""
    csr = as_csr(matrix)
    n = csr.shape[0]
    idx = range(n_vec) if indices is None else indices
    quads, facts = [], []
    for l in idx:
        a, b, bn, _, _ = lanczos_factorize(csr, draw_probe(kind, seed, n, l), steps, reorth)
        facts.append((a, b, bn))
        quads.append(ritz_quadrature(a, b))
    theta, tau = pool(quads)
    return blur_nodes(theta, tau, grid, sigma), theta, tau, facts


# ---- Gershgorin (configs) ---------------------------------------------------------------------
def gershgorin(csr):
    n = csr.shape[0]
    rows = np.repeat(np.arange(n), np.diff(csr.indptr))
    on = rows == csr.indices
    dg = np.bincount(rows[on], weights=csr.data[on], minlength=n)
    rad = np.bincount(rows[~on], weights=np.abs(csr.data[~on]), minlength=n)
    return float(np.min(dg - rad)), float(np.max(dg + rad))


# ---- lanczos.py:162-167, matrix.py:207-241 (spectral-interval estimation) -----------------------
def ritz_residual_bounds(alpha, beta, beta_next):
    if len(alpha) == 1:
        return alpha.copy(), np.array([abs(beta_next)])
    theta, y = eigh_tridiagonal(alpha, beta)
    return theta, abs(beta_next) * np.abs(y[-1, :])


def estimate_spectral_interval(matrix, lanczos_steps=20, margin=0.01, seed=0):
    """(lb, ub) after widening: extreme Ritz values -/+ residual bounds (matrix.py:207-241)."""
    csr = as_csr(matrix)
    n = csr.shape[0]
    steps = min(lanczos_steps, n)
    v0 = draw_probe("gaussian", seed, n, 0, stream=0xB0)
    if np.linalg.norm(v0) == 0.0:
        v0 = draw_probe("gaussian", seed, n, 1, stream=0xB0)
    alpha, beta, beta_next, _, _ = lanczos_factorize(csr, v0, steps)
    theta, resid = ritz_residual_bounds(alpha, beta, beta_next)
    lb = theta[0] - resid[0]
    ub = theta[-1] + resid[-1]
    if ub <= lb:
        half = max(abs(ub), 1.0) * 1e-8
        lb, ub = lb - half, ub + half
    c, h = 0.5 * (lb + ub), (1.0 + margin) * (0.5 * (ub - lb))  # SpectralInterval.widened (density.py:43-46)
    return c - h, c + h


# ---- lanczos.py:222-293 (Haydock resolvent) ------------------------------------------------------
def continued_fraction_resolvent(alpha, beta, z):
    z = np.asarray(z, dtype=complex)
    f = 1.0 / (z - alpha[-1])
    for j in range(len(alpha) - 2, -1, -1):
        f = 1.0 / (z - alpha[j] - beta[j] ** 2 * f)
    return f


def tridiagonal_resolvent_first(alpha, beta, z):
    z = np.asarray(z, dtype=complex)
    m = len(alpha)
    if m == 1:
        w = 1.0 / (z - alpha[0])
        return w, w
    cp = np.empty((m - 1,) + z.shape, dtype=complex)
    dp = np.empty((m,) + z.shape, dtype=complex)
    denom = z - alpha[0]
    cp[0] = -beta[0] / denom
    dp[0] = 1.0 / denom
    for j in range(1, m):
        denom = (z - alpha[j]) + beta[j - 1] * cp[j - 1]
        if j < m - 1:
            cp[j] = -beta[j] / denom
        dp[j] = beta[j - 1] * dp[j - 1] / denom
    w = dp[m - 1]
    w_last = w
    for j in range(m - 2, -1, -1):
        w = dp[j] - cp[j] * w
    return w, w_last


def haydock_dos(matrix, steps, kind, seed, n_vec, eta, grid, reorth="full"):
    """(density, truncation_indicator) on the original-coordinate grid."""
    csr = as_csr(matrix)
    z = np.asarray(grid, dtype=float) + 1j * eta
    dens, trunc = [], []
    for l in range(n_vec):
        a, b, bn, _, _ = lanczos_factorize(csr, draw_probe(kind, seed, csr.shape[0], l), steps, reorth)
        f = continued_fraction_resolvent(a, b, z)
        _, w_last = tridiagonal_resolvent_first(a, b, z)
        dens.append(-np.imag(f) / np.pi)
        trunc.append(bn * float(np.max(np.abs(w_last))))
    return np.mean(dens, axis=0), max(trunc)


# ---- dgl.py:35-132 (Delta-Gauss-Legendre) ---------------------------------------------------------
def dgl_gamma_table(t, sigma, max_degree, tol=1e-6):
    """(gamma, psi, effective) for centres t (dgl.py:42-89)."""
    from scipy.special import erf

    t = np.asarray(t, dtype=float)
    gamma = np.zeros((max_degree + 1, t.size))
    psi = np.zeros((max_degree + 1, t.size))
    s = np.sqrt(2.0) * sigma
    gamma[0] = sigma * np.sqrt(np.pi / 2.0) * (erf((1.0 - t) / s) + erf((1.0 + t) / s))
    effective = np.full(t.size, max_degree)
    active = np.ones(t.size, dtype=bool)
    exp_lo = np.exp(-0.5 * ((1.0 - t) / sigma) ** 2)
    exp_hi = np.exp(-0.5 * ((1.0 + t) / sigma) ** 2)
    psi_k = np.zeros(t.size)
    psi_next = gamma[0].copy()
    if max_degree >= 1:
        psi[1] = psi_next
    for k in range(max_degree):
        if k >= 1:
            halted = active & (np.abs(gamma[k - 1]) + np.abs(gamma[k]) <= k * tol)
            effective[halted] = k
            active &= ~halted
            if not active.any():
                break
        boundary_term = exp_lo - (-1.0) ** k * exp_hi
        gamma_prev = gamma[k - 1] if k >= 1 else 0.0
        nxt = ((2 * k + 1) / (k + 1.0) * (sigma * sigma * (psi_k - boundary_term) + t * gamma[k])
               - k / (k + 1.0) * gamma_prev)
        gamma[k + 1, active] = nxt[active]
        j = k + 1
        psi_k, psi_next = psi_next, (2 * j + 1) * gamma[j] + psi_k
        if j + 1 <= max_degree:
            psi[j + 1, active] = psi_next[active]
    return gamma, psi, effective


def dgl_dos(zeta, n, d, sigma, t, tol=1e-6):
    """(values, density) of evaluate_dgl_dos (dgl.py:109-132); sigma in original units."""
    sigma_m = sigma / d
    gamma, _, _ = dgl_gamma_table(t, sigma_m, len(zeta) - 1, tol)
    k = np.arange(len(zeta))
    values = (((k + 0.5) * zeta) @ gamma) / (n * np.sqrt(2.0 * np.pi) * sigma_m)
    return values, values / d

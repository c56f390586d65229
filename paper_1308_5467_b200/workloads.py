"""Synthetic matrices of BASELINE.json's five configs (seeded, deterministic).

The reference measures on nothing but these shapes: there is no
public benchmark suite, so seeded generators with the named sizes and value
distributions are the workload.

  C1  generate_modified_laplacian_2d(100, 100, bumps=())  (matrix.py:173-204)
  C2  Anderson model, 7-point periodic 64^3, V ~ U[-W/2, W/2], W = 16.5, rng(2)
  C3  n = 1e6 band |i-j| <= 20 + 10 random upper off-band entries per row,
      mirrored; off-diagonals N(0,1)/sqrt(60), diagonal U[-2, 2], rng(3)
  C4  Lanczos on the C2 matrix
  C5  27-point periodic 256^3, 13 independent weights U[-1,1] mirrored,
      centre U[-1,1], diagonal centre + V, V ~ U[-1,1], rng(5)

Spectral intervals come from Gershgorin discs (BASELINE.json asks for
Gershgorin bounds; the reference only has Lanczos bounds, matrix.py:207-241).
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .density import SpectralInterval
from .operators import SparseSymmetricMatrix, StencilOperator


# ---------------------------------------------------------------------------
# C1: the reference's model problem, built directly as sorted int32 CSR


# the reference's frozen test potential (matrix.py:24-29): a shallow well at
# (4, 5) and a sharp barrier at (25, 15)
DEFAULT_BUMPS = ((4.0, 5.0, -0.13, 4.0), (25.0, 15.0, 5.0, 1.5))


def generate_modified_laplacian_2d(nx, ny, bumps=DEFAULT_BUMPS):
    """5-point Dirichlet Laplacian plus Gaussian bumps (matrix.py:173-204).

    Builds the CSR the reference produces (diagonal 4 + potential, off-
    diagonals -1, columns sorted) without the kron/symmetrise detour; tests
    pin it bit-for-bit against the reference when that is importable.
    """
    if nx < 1 or ny < 1:
        raise ValueError("grid must have at least one point per dimension")
    n = nx * ny
    p = np.arange(n, dtype=np.int64)
    i, j = p % nx, p // nx
    x = np.arange(1, nx + 1, dtype=float)
    y = np.arange(1, ny + 1, dtype=float)
    xx, yy = np.meshgrid(x, y)
    v = np.zeros(n)
    for cx, cy, height, width in bumps:
        if width <= 0:
            raise ValueError("bump width must be positive")
        r2 = (xx - cx) ** 2 + (yy - cy) ** 2
        v += (height * np.exp(-r2 / (2.0 * width**2))).ravel()
    diag = 4.0 + v
    # candidate columns in increasing order: p-nx, p-1, p, p+1, p+nx
    cols = np.stack([p - nx, p - 1, p, p + 1, p + nx], axis=1)
    vals = np.stack([np.full(n, -1.0), np.full(n, -1.0), diag, np.full(n, -1.0), np.full(n, -1.0)], axis=1)
    keep = np.stack([j > 0, i > 0, np.ones(n, bool), i < nx - 1, j < ny - 1], axis=1)
    if nx == 1:
        keep[:, 1] = keep[:, 3] = False
    if ny == 1:
        keep[:, 0] = keep[:, 4] = False
    counts = keep.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    # the reference symmetrises as (a + a.T) * 0.5, which is exact here
    vals = (vals + vals) * 0.5
    csr = sp.csr_array((vals[keep], cols[keep].astype(np.int32), indptr.astype(np.int32)), shape=(n, n))
    return SparseSymmetricMatrix(csr=csr)


# ---------------------------------------------------------------------------
# structured configs as stencils (C2, C5)

FACE_OFFSETS = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]


def anderson_3d(L=64, W=16.5, seed=2):
    """7-point periodic Laplacian (6I - adjacency) + V, V ~ U[-W/2, W/2]."""
    rng = np.random.default_rng(seed)
    n = L * L * L
    pot = rng.uniform(-W / 2.0, W / 2.0, n)
    return StencilOperator((L, L, L), FACE_OFFSETS, [-1.0] * 6, 6.0 + pot)


def _positive_offsets_27():
    """The 13 lexicographically positive offsets of the 3x3x3 cube."""
    out = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if (dz, dy, dx) > (0, 0, 0):
                    out.append((dx, dy, dz))
    return out


def stencil27_3d(L=256, seed=5):
    """27-point periodic stencil: symmetric weights U[-1,1], diag = w0 + V."""
    rng = np.random.default_rng(seed)
    pos = _positive_offsets_27()
    wpos = rng.uniform(-1.0, 1.0, len(pos))
    w0 = rng.uniform(-1.0, 1.0)
    n = L * L * L
    pot = rng.uniform(-1.0, 1.0, n)
    offsets, weights = [], []
    for o, w in zip(pos, wpos):
        offsets.append(o)
        weights.append(float(w))
        offsets.append((-o[0], -o[1], -o[2]))
        weights.append(float(w))
    return StencilOperator((L, L, L), offsets, weights, w0 + pot)


# ---------------------------------------------------------------------------
# C3: band + random off-band, pattern and values mirrored bit-exactly


def dft_like(n=1_000_000, half_band=20, n_random=10, seed=3, scale_nnz=60.0):
    """Band of half-width 20 plus random off-band couplings, symmetric.

    Every row draws ``n_random`` columns uniformly among its off-band
    columns; each drawn pair (i, j) is stored once in the upper triangle
    (duplicates removed explicitly) and mirrored, so a row carries about
    2 * n_random off-band entries (~61 nnz/row at the default).  Values:
    band and off-band N(0,1)/sqrt(60), mirrored bit-exactly; diagonal
    U[-2, 2].  Draw order: diagonal, band (by offset), columns, values.
    """
    rng = np.random.default_rng(seed)
    sdev = 1.0 / np.sqrt(scale_nnz)
    diag = rng.uniform(-2.0, 2.0, n)
    rows_parts, cols_parts, vals_parts = [], [], []
    for k in range(1, half_band + 1):
        i = np.arange(0, n - k, dtype=np.int64)
        rows_parts.append(i)
        cols_parts.append(i + k)
        vals_parts.append(rng.standard_normal(n - k) * sdev)
    i = np.repeat(np.arange(n, dtype=np.int64), n_random)
    lo_b = np.maximum(i - half_band, 0)
    hi_b = np.minimum(i + half_band, n - 1)
    nb = hi_b - lo_b + 1
    avail = n - nb
    u = rng.random(i.size)
    j = np.floor(u * avail).astype(np.int64)
    j += (j >= lo_b) * nb
    ok = avail > 0
    i, j = i[ok], j[ok]
    key = np.unique(np.minimum(i, j) * n + np.maximum(i, j))  # upper-triangle pairs, deduplicated
    i, j = key // n, key % n
    rows_parts.append(i)
    cols_parts.append(j)
    vals_parts.append(rng.standard_normal(i.size) * sdev)
    ur = np.concatenate(rows_parts)
    uc = np.concatenate(cols_parts)
    uv = np.concatenate(vals_parts)
    ar = np.arange(n, dtype=np.int64)
    rows = np.concatenate([ur, uc, ar])
    cols = np.concatenate([uc, ur, ar]).astype(np.int32)
    vals = np.concatenate([uv, uv, diag])
    coo = sp.coo_array((vals, (rows.astype(np.int32), cols)), shape=(n, n))
    csr = sp.csr_array(coo.tocsr())
    csr.sort_indices()
    csr.indptr = csr.indptr.astype(np.int64)
    return SparseSymmetricMatrix(csr=csr)


# ---------------------------------------------------------------------------
# Gershgorin bounds


def gershgorin_interval(op):
    """[min(a_ii - R_i), max(a_ii + R_i)], R_i = sum_{j != i} |a_ij|."""
    if isinstance(op, StencilOperator):
        r = float(np.sum(np.abs(op.weights)))
        return SpectralInterval(float(op.diag.min()) - r, float(op.diag.max()) + r)
    csr = op.csr if hasattr(op, "csr") else sp.csr_array(op)
    n = csr.shape[0]
    rows = np.repeat(np.arange(n), np.diff(csr.indptr))
    on = rows == csr.indices
    dg = np.bincount(rows[on], weights=csr.data[on], minlength=n)
    rad = np.bincount(rows[~on], weights=np.abs(csr.data[~on]), minlength=n)
    return SpectralInterval(float(np.min(dg - rad)), float(np.max(dg + rad)))


# ---------------------------------------------------------------------------
# the five configs


@dataclass
class Config:
    name: str
    method: str            # "kpm-jackson" or "lanczos"
    degree: int            # M (moments) or Lanczos steps
    n_vec: int
    probe_kind: str
    grid_points: int
    sigma: float = None
    description: str = ""


CONFIGS = {
    "C1": Config("C1", "kpm-jackson", 100, 20, "gaussian", 1000,
                 description="2D 5-point Laplacian 100x100, KPM M=100, 20 Gaussian probes, 1000 pts"),
    "C2": Config("C2", "kpm-jackson", 500, 64, "rademacher", 2000,
                 description="3D Anderson 64^3 W=16.5, KPM M=500, 64 Rademacher probes, 2000 pts"),
    "C3": Config("C3", "kpm-jackson", 1000, 128, "gaussian", 2000,
                 description="synthetic DFT-like n=1e6 ~61 nnz/row, KPM M=1000, 128 Gaussian probes"),
    "C4": Config("C4", "lanczos", 100, 128, "gaussian", 2000, sigma=0.01,
                 description="Lanczos m=100 full reorth on the C2 matrix, 128 Gaussian probes, sigma=0.01"),
    "C5": Config("C5", "kpm-jackson", 2000, 32, "rademacher", 2000,
                 description="27-point periodic stencil 256^3, KPM M=2000, 32 Rademacher probes"),
}


def build_matrix(name, scale=1.0):
    """Matrix object of a config; ``scale`` < 1 shrinks the grid for tests."""
    if name == "C1":
        return generate_modified_laplacian_2d(100, 100, bumps=())
    if name in ("C2", "C4"):
        L = max(4, int(round(64 * scale)))
        return anderson_3d(L)
    if name == "C3":
        return dft_like(max(1000, int(1_000_000 * scale)))
    if name == "C5":
        L = max(4, int(round(256 * scale)))
        return stencil27_3d(L)
    raise KeyError(name)

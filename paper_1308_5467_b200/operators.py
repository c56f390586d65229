"""The operator side of the drop-in boundary.

The reference's plugin API is duck-typed: "anything with a ``dim`` attribute
and a ``matvec(x)`` method" (specdens/matrix.py:3-6).  Its front door wraps the
matrix as ``MappedOperator(MatvecCounter(SparseSymmetricMatrix))``
(compare.py:93-96).  The GPU engine never calls ``matvec``: it walks that
chain, reads the affine map (c, d) from every ``MappedOperator`` and the CSR
arrays (or the stencil description) from the innermost matrix, uploads them
once to a device handle, and adds the analytic MATVEC count to every
``MatvecCounter`` it passed.  Objects that expose only ``matvec`` cannot be
offloaded and raise ``TypeError`` (there is no CPU fallback).

The classes below mirror the reference's (matrix.py:35-170) so code written
against ``specdens`` finds the same names; the reference's own instances are
accepted as well.  Their ``matvec`` methods exist only for interop with code
that calls the protocol directly; the engine does not use them.
"""

import ctypes
import os
import threading
import weakref
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native


# ---------------------------------------------------------------------------
# host-side operator types (mirrors of matrix.py:35-170)


@dataclass
class SparseSymmetricMatrix:
    """Real symmetric CSR matrix, both triangles stored (matrix.py:35-109)."""

    csr: sp.csr_array
    symmetric_storage: bool = False

    @classmethod
    def from_coo(cls, n, rows, cols, vals, symmetric_storage=False):
        """CSR from coordinate triplets with duplicates summed (contract of
        matrix.py:47-70): one stored triangle is mirrored when
        ``symmetric_storage`` is set, otherwise the triplets must already
        describe an exactly symmetric matrix."""
        i, j = (np.asarray(x, dtype=np.int64) for x in (rows, cols))
        v = np.asarray(vals, dtype=np.float64)
        for idx in (i, j):
            if idx.size and not (0 <= idx.min() and idx.max() < n):
                raise ValueError("coordinate index out of range")
        if symmetric_storage:  # append the transposed strict triangle after the given entries
            strict = np.flatnonzero(i != j)
            i, j, v = np.r_[i, j[strict]], np.r_[j, i[strict]], np.r_[v, v[strict]]
        csr = sp.coo_array((v, (i, j)), shape=(n, n)).tocsr()
        csr.sum_duplicates()
        out = cls(csr=csr, symmetric_storage=symmetric_storage)
        if not out.is_symmetric():
            raise ValueError("matrix data is not symmetric")
        return out

    @classmethod
    def from_dense(cls, a):
        """CSR of an exactly symmetric dense array (matrix.py:72-79)."""
        dense = np.asarray(a, dtype=float)
        if dense.ndim != 2 or dense.shape[0] != dense.shape[1]:
            raise ValueError("dense input must be square")
        if (dense != dense.T).any():
            raise ValueError("dense input must be exactly symmetric")
        return cls(csr=sp.csr_array(dense))

    @property
    def n(self):
        return self.csr.shape[0]

    @property
    def dim(self):
        return self.csr.shape[0]

    def matvec(self, x):  # interop only; the engine never calls it
        return self.csr @ x

    def is_symmetric(self):
        return (self.csr != self.csr.T).nnz == 0


class StencilOperator:
    """Periodic constant-coefficient stencil on an nx*ny*nz grid (nx fastest).

    (A x)_p = diag[p] x_p + sum_o weights[o] x_{p + offsets[o]} with periodic
    wrap.  Not a reference type: it is the matrix-free form of the structured
    configs (Anderson 7-point, 27-point), satisfies the same protocol, and
    exposes ``csr`` (built lazily) so the CPU oracle and the reference can run
    on exactly the same operator.
    """

    z_ghost = False  # see SlabStencil

    def __init__(self, shape, offsets, weights, diag):
        self.shape = tuple(int(s) for s in shape)
        if len(self.shape) != 3 or min(self.shape) < 1:
            raise ValueError("stencil shape must be three positive extents (nx, ny, nz)")
        self.offsets = [tuple(int(v) for v in o) for o in offsets]
        self.weights = [float(w) for w in weights]
        if len(self.offsets) != len(self.weights) or len(self.offsets) > 26:
            raise ValueError("need one weight per offset, at most 26 off-centre points")
        for o in self.offsets:
            if len(o) != 3 or any(abs(v) > 1 for v in o) or o == (0, 0, 0):
                raise ValueError(f"bad stencil offset {o}")
        if len(set(self.offsets)) != len(self.offsets):
            raise ValueError("duplicate stencil offsets")
        self.diag = np.ascontiguousarray(diag, dtype=np.float64)
        nx, ny, nz = self.shape
        if self.diag.shape != (nx * ny * nz,):
            raise ValueError("diag must have one entry per grid point")
        # a stencil offset and its wrap-around image must differ, else the
        # CSR form would merge entries (needs extent >= 3 along moved axes)
        for axis in range(3):
            if any(o[axis] != 0 for o in self.offsets) and self.shape[axis] < 3:
                raise ValueError("periodic stencils need at least 3 points along every coupled axis")
        self._csr = None

    @property
    def dim(self):
        return int(self.diag.shape[0])

    @property
    def n(self):
        return self.dim

    @property
    def nnz(self):
        return self.dim * (len(self.offsets) + 1)

    @property
    def csr(self):
        """The same operator as a sorted-column CSR array (both triangles)."""
        if self._csr is None:
            nx, ny, nz = self.shape
            n = self.dim
            p = np.arange(n, dtype=np.int64)
            ix, iy, iz = p % nx, (p // nx) % ny, p // (nx * ny)
            cols = [p]
            vals = [self.diag]
            for (dx, dy, dz), w in zip(self.offsets, self.weights):
                jx, jy, jz = (ix + dx) % nx, (iy + dy) % ny, (iz + dz) % nz
                cols.append((jz * ny + jy) * nx + jx)
                vals.append(np.full(n, w))
            cols = np.stack(cols, axis=1)
            vals = np.stack(vals, axis=1)
            order = np.argsort(cols, axis=1, kind="stable")
            cols = np.take_along_axis(cols, order, axis=1)
            vals = np.take_along_axis(vals, order, axis=1)
            k = cols.shape[1]
            indptr = np.arange(0, n * k + 1, k, dtype=np.int64)
            self._csr = sp.csr_array((vals.ravel(), cols.ravel().astype(np.int32), indptr), shape=(n, n))
        return self._csr

    def matvec(self, x):  # interop only; the engine never calls it
        return self.csr @ x


class SlabStencil(StencilOperator):
    """Planes [z0, z1) of a periodic StencilOperator, for the row partition.

    The slab's operator is not periodic in z: the neighbours of its first and
    last plane live in ghost planes that the caller keeps immediately before
    and after the slab's rows in every block (sdb_stencil_desc.z_ghost).
    """

    z_ghost = True

    def __init__(self, parent, z0, z1):
        nx, ny, nz = parent.shape
        if not (0 <= z0 < z1 <= nz):
            raise ValueError(f"bad slab [{z0}, {z1}) of {nz} planes")
        self.parent = parent
        self.z0, self.z1 = int(z0), int(z1)
        self.shape = (nx, ny, self.z1 - self.z0)
        self.offsets = list(parent.offsets)
        self.weights = list(parent.weights)
        self.diag = np.ascontiguousarray(parent.diag[self.z0 * nx * ny:self.z1 * nx * ny])
        self._csr = None

    @property
    def csr(self):
        raise TypeError("a slab has no standalone CSR form (its z neighbours live on other ranks)")

    def matvec(self, x):
        raise TypeError("a slab has no standalone matvec")


class MappedOperator:
    """B = (A - cI)/d of an operator onto the unit interval (matrix.py:112-126)."""

    def __init__(self, op, interval):
        self.op = op
        self.interval = interval
        self.c = interval.center
        self.d = interval.halfwidth

    @property
    def dim(self):
        return self.op.dim

    def matvec(self, x):  # interop only
        return (self.op.matvec(x) - self.c * x) / self.d


class MatvecCounter:
    """Counts MATVECs (matrix.py:129-142); the engine adds analytic counts."""

    def __init__(self, op):
        self.op = op
        self.count = 0

    @property
    def dim(self):
        return self.op.dim

    def matvec(self, x):  # interop only
        self.count += 1
        return self.op.matvec(x)


class _DenseOperator:
    def __init__(self, a):
        self.a = np.asarray(a, dtype=float)
        self.dim = self.a.shape[0]

    def matvec(self, x):  # interop only
        return self.a @ x

    def toarray(self):
        return self.a


def as_operator(obj):
    """Adapt a matrix-like object to the operator protocol (matrix.py:157-165)."""
    if hasattr(obj, "matvec") and hasattr(obj, "dim"):
        return obj
    if isinstance(obj, np.ndarray):
        return _DenseOperator(obj)
    if sp.issparse(obj):
        return SparseSymmetricMatrix(csr=sp.csr_array(obj))
    raise TypeError(f"cannot interpret {type(obj).__name__} as a linear operator")


def apply_spectral_map(op, interval):
    """(A - cI)/d without copying the matrix (matrix.py:168-170)."""
    return MappedOperator(as_operator(op), interval)


# ---------------------------------------------------------------------------
# operator chain -> device handle


@dataclass
class ResolvedOperator:
    """What the engine needs from an operator chain."""

    base: object          # innermost matrix-like object
    c: float              # B = (A - c I) / d
    d: float
    counters: list        # MatvecCounter-like objects to credit
    dim: int


def resolve(op):
    """Walk MappedOperator / MatvecCounter wrappers down to the matrix.

    Nested maps compose: ((A - c1)/d1 - c2)/d2 = (A - (c1 + c2 d1)) / (d1 d2).
    """
    c, d = 0.0, 1.0
    counters = []
    obj = op
    seen = 0
    while True:
        seen += 1
        if seen > 64:
            raise TypeError("operator chain too deep")
        if _is_mapped(obj):
            c_i, d_i = float(obj.c), float(obj.d)
            # running map (X - c)/d with X = (A' - c_i)/d_i underneath
            c, d = c_i + c * d_i, d * d_i
            obj = obj.op
            continue
        if _is_counter(obj):
            counters.append(obj)
            obj = obj.op
            continue
        break
    base = _base_matrix(obj)
    dim = int(base.dim) if hasattr(base, "dim") else int(base.shape[0])
    return ResolvedOperator(base=base, c=c, d=d, counters=counters, dim=dim)


def _is_mapped(obj):
    return hasattr(obj, "op") and hasattr(obj, "c") and hasattr(obj, "d") and hasattr(obj, "matvec")


def _is_counter(obj):
    return hasattr(obj, "op") and hasattr(obj, "count") and hasattr(obj, "matvec") and not _is_mapped(obj)


def _base_matrix(obj):
    if isinstance(obj, StencilOperator):
        return obj
    if hasattr(obj, "csr") and sp.issparse(getattr(obj, "csr")):
        return obj
    if isinstance(obj, np.ndarray):
        return _DenseOperator(obj)
    if hasattr(obj, "a") and isinstance(getattr(obj, "a"), np.ndarray) and hasattr(obj, "matvec"):
        return obj  # reference _DenseOperator
    if sp.issparse(obj):
        return SparseSymmetricMatrix(csr=sp.csr_array(obj))
    raise TypeError(
        f"cannot offload operator of type {type(obj).__name__} to the GPU: it exposes no CSR "
        "arrays or stencil description (only matvec); there is no CPU fallback"
    )


def _csr_arrays(base):
    if hasattr(base, "csr"):
        csr = base.csr
    else:
        csr = sp.csr_array(np.asarray(base.a, dtype=float))
    if not isinstance(csr, (sp.csr_array, sp.csr_matrix)):
        csr = sp.csr_array(csr)
    n = csr.shape[0]
    if csr.shape[0] != csr.shape[1]:
        raise ValueError("matrix must be square")
    return csr, n


def _divisors(v, lo=3):
    out = []
    i = 1
    while i * i <= v:
        if v % i == 0:
            for d in (i, v // i):
                if d >= lo and d not in out:
                    out.append(d)
        i += 1
    return sorted(out)


def detect_stencil(csr):
    """Recognise a CSR that is exactly a periodic constant-coefficient stencil.

    Part of the matrix layer's format selection: when every row stores the
    same pattern of <= 27 neighbours on some nx*ny*nz torus (nx, ny, nz >= 3)
    with one constant weight per neighbour offset, the matrix is re-expressed
    as a ``StencilOperator`` with the CSR's own diagonal -- the identical
    operator, whose step kernels gather neighbours by index arithmetic
    instead of streaming column indices.  The candidate is accepted only if
    its CSR form equals the input array for array (indices and values).
    Returns None otherwise.
    """
    n = csr.shape[0]
    if n < 27:
        return None
    counts = np.diff(csr.indptr)
    k = int(counts[0])
    if k < 2 or k > 27 or np.any(counts != k):
        return None
    if not csr.has_sorted_indices:
        return None
    cols = np.asarray(csr.indices).reshape(n, k)
    vals = np.asarray(csr.data).reshape(n, k)
    for nx in _divisors(n):
        for ny in _divisors(n // nx):
            nz = n // (nx * ny)
            if nz < 3:
                continue
            r = ((nz // 2) * ny + ny // 2) * nx + nx // 2
            d = cols[r].astype(np.int64) - r
            offs, weights, has_diag = [], [], False
            ok = True
            for dd, vv in zip(d, vals[r]):
                dz = int(np.round(dd / (nx * ny)))
                rem = dd - dz * nx * ny
                dy = int(np.round(rem / nx))
                dx = int(rem - dy * nx)
                if max(abs(dx), abs(dy), abs(dz)) > 1:
                    ok = False
                    break
                if dx == dy == dz == 0:
                    has_diag = True
                else:
                    offs.append((dx, dy, dz))
                    weights.append(float(vv))
            if not ok or not has_diag or not offs:
                continue
            on = cols == np.arange(n)[:, None]
            if not np.all(on.sum(axis=1) == 1):
                return None
            diag = np.ascontiguousarray(vals[on], dtype=np.float64)
            try:
                cand = StencilOperator((nx, ny, nz), offs, weights, diag)
            except ValueError:
                continue
            ref = cand.csr
            if np.array_equal(ref.indices, csr.indices) and np.array_equal(ref.data, csr.data):
                return cand
    return None


class DeviceMatrix:
    """Owns one ``sdb_matrix`` handle on one CUDA device."""

    def __init__(self, handle, device, n, nnz, fmt, stream_bytes, detected=False):
        self.detected_stencil = detected  # CSR input re-expressed as a stencil
        self.handle = handle
        self.device = device
        self.n = n
        self.nnz = nnz
        self.format = fmt
        self.bytes_per_pass = stream_bytes  # M_A: matrix bytes one SpMM streams
        self.band_half_width = 0
        self.band_far_entries = 0
        self.band_bytes_per_pass = 0
        self._finalizer = weakref.finalize(self, _destroy_handle, handle)

    @classmethod
    def upload(cls, base, device, stream, auto_stencil=None):
        if auto_stencil is None:
            auto_stencil = auto_stencil_enabled()
        lib = _native.load()
        h = ctypes.c_void_p()
        if isinstance(base, StencilOperator):
            desc = _native.SdbStencilDesc()
            desc.nx, desc.ny, desc.nz = base.shape
            desc.n_offsets = len(base.offsets)
            desc.z_ghost = 1 if getattr(base, "z_ghost", False) else 0
            for i, (o, w) in enumerate(zip(base.offsets, base.weights)):
                for a in range(3):
                    desc.offsets[i][a] = o[a]
                desc.weights[i] = w
            diag = np.ascontiguousarray(base.diag, dtype=np.float64)
            _native.check(lib.sdb_matrix_create_stencil(device, ctypes.byref(desc), diag.ctypes.data,
                                                        stream, ctypes.byref(h)))
        elif auto_stencil and (st := detect_stencil(_csr_arrays(base)[0])) is not None:
            dm = cls.upload(st, device, stream, auto_stencil=False)
            dm.detected_stencil = True
            return dm
        else:
            csr, n = _csr_arrays(base)
            indptr = np.ascontiguousarray(csr.indptr, dtype=np.int64)
            idx = csr.indices
            if idx.dtype == np.int32:
                bits = 32
                idx = np.ascontiguousarray(idx)
            else:
                bits = 64
                idx = np.ascontiguousarray(idx, dtype=np.int64)
            data = np.ascontiguousarray(csr.data, dtype=np.float64)
            _native.check(lib.sdb_matrix_create_csr(device, n, int(indptr[-1]), indptr.ctypes.data,
                                                    idx.ctypes.data if idx.size else None, bits,
                                                    data.ctypes.data if data.size else None, stream,
                                                    ctypes.byref(h)))
        info = _native.SdbMatrixInfo()
        _native.check(lib.sdb_matrix_get_info(h, ctypes.byref(info)))
        dm = cls(h, device, info.n, info.nnz, info.format, info.bytes)
        hb, far, bpp = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        _native.check(lib.sdb_matrix_band_info(h, ctypes.byref(hb), ctypes.byref(far), ctypes.byref(bpp)))
        dm.band_half_width = hb.value    # dense-band + far split (band.cu); 0: plain CSR
        dm.band_far_entries = far.value
        dm.band_bytes_per_pass = bpp.value  # matrix bytes one 16-probe slice pass streams
        return dm


def _destroy_handle(h):
    try:
        _native.load().sdb_matrix_destroy(h)
    except Exception:  # interpreter shutdown
        pass


# Cache of device handles keyed by the identity of the host matrix object.
# Operators are immutable by contract ("SparseSymmetricMatrix
# is immutable after construction"), so a handle stays valid as long as the
# host object lives; the entry dies with it.
_cache_lock = threading.Lock()
_cache = {}


def auto_stencil_enabled():
    """CSR -> stencil format selection (SDB_AUTO_STENCIL=0 disables it)."""
    return os.environ.get("SDB_AUTO_STENCIL", "1") != "0"


def _cache_key(base, device):
    if isinstance(base, StencilOperator):
        arr = base.diag
        return (id(base), device, arr.ctypes.data, arr.shape[0], "stencil")
    csr = base.csr if hasattr(base, "csr") else None
    if csr is not None:
        return (id(base), device, csr.data.ctypes.data, csr.indices.ctypes.data, csr.nnz, "csr",
                auto_stencil_enabled())
    return None


def device_matrix(base, device, stream):
    """Device handle for a resolved base matrix (cached per host object)."""
    key = _cache_key(base, device)
    if key is None:
        return DeviceMatrix.upload(base, device, stream)
    with _cache_lock:
        ent = _cache.get(key)
        if ent is not None:
            ref, dm = ent
            if ref() is base:
                return dm
    dm = DeviceMatrix.upload(base, device, stream)
    try:
        ref = weakref.ref(base, lambda _r, k=key: _drop(k))
    except TypeError:  # not weak-referenceable: do not cache
        return dm
    with _cache_lock:
        _cache[key] = (ref, dm)
    return dm


def _drop(key):
    with _cache_lock:
        _cache.pop(key, None)


def clear_device_cache():
    with _cache_lock:
        _cache.clear()


# ---------------------------------------------------------------------------
# Spectral-interval estimation (matrix.py:207-241): the
# 20-step Lanczos run and the residual-bounded Ritz extremes on the device.

DEFAULT_LANCZOS_STEPS = 20
DEFAULT_INTERVAL_MARGIN = 0.01


def estimate_spectral_interval(op, lanczos_steps=DEFAULT_LANCZOS_STEPS, margin=DEFAULT_INTERVAL_MARGIN, v0=None,
                               seed=0, device=None):
    """Lanczos-based eigenvalue bounds, widened by a relative safety margin.

    Same contract as the reference: ``lanczos_steps`` iterations from a
    Gaussian probe on the reserved stream, extreme Ritz values -/+ their
    residual bounds, a zero start vector resampled once, non-finite bounds ->
    NumericalFailure, a single-point spectrum opened by 1e-8 max(|ub|, 1).
    """
    from .density import SpectralInterval
    from .errors import NumericalFailure
    from .lanczos import lanczos_factorize, ritz_residual_bounds
    from .stochastic import INTERVAL_STREAM, ProbeVectorSource

    if lanczos_steps < 2:
        raise ValueError("interval estimation needs at least 2 Lanczos steps")
    op = as_operator(op)
    steps = min(lanczos_steps, op.dim)
    src = ProbeVectorSource("gaussian", seed=seed, dim=op.dim, stream=INTERVAL_STREAM)
    if v0 is None:
        v0 = src.draw(0)
    v0 = np.asarray(v0, dtype=float)
    if np.linalg.norm(v0) == 0.0:
        v0 = src.draw(1)
        if np.linalg.norm(v0) == 0.0:
            raise NumericalFailure("starting vector for interval estimation is zero")
    fact = lanczos_factorize(op, v0, steps, device=device)
    theta, resid = ritz_residual_bounds(fact, device=device)
    lb = theta[0] - resid[0]
    ub = theta[-1] + resid[-1]
    if not np.isfinite(lb) or not np.isfinite(ub):
        raise NumericalFailure("non-finite eigenvalue bounds")
    if ub <= lb:
        half = max(abs(ub), 1.0) * 1e-8
        lb, ub = lb - half, ub + half
    return SpectralInterval(lb, ub).widened(margin)


# ---------------------------------------------------------------------------
# Matrix Market coordinate IO (matrix.py:247-331): the reader
# is native (libspecdens_b200 ``sdb_mm_read``: parse, expand, sum duplicates,
# exact symmetry check); the matrix then uploads to the device like any CSR.


def load_matrix_market(path):
    """Read a real coordinate Matrix Market file into a SparseSymmetricMatrix
    (same accepted headers, expansion, duplicate summing and ValueErrors as
    matrix.py:247-304)."""
    lib = _native.load()
    h = ctypes.c_void_p()
    _native.check(lib.sdb_mm_read(os.fsencode(str(path)), ctypes.byref(h)))
    try:
        n, nnz, sym = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        _native.check(lib.sdb_mm_info(h, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(sym)))
        indptr = np.empty(n.value + 1, dtype=np.int64)
        indices = np.empty(nnz.value, dtype=np.int32)
        data = np.empty(nnz.value, dtype=np.float64)
        _native.check(lib.sdb_mm_export(h, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data))
    finally:
        lib.sdb_mm_free(h)
    if nnz.value < 2**31 - 1:  # SciPy wants one index dtype for indptr and indices
        indptr = indptr.astype(np.int32)
    else:
        indices = indices.astype(np.int64)
    csr = sp.csr_array((data, indices, indptr), shape=(n.value, n.value))
    return SparseSymmetricMatrix(csr=csr, symmetric_storage=bool(sym.value))


def save_matrix_market(mat, path):
    """Write the lower triangle as a real symmetric coordinate file (matrix.py:321-331)."""
    coo = sp.tril(mat.csr).tocoo()
    with open(path, "w", encoding="ascii") as fh:
        fh.write("%%MatrixMarket matrix coordinate real symmetric\n")
        fh.write(f"{mat.n} {mat.n} {coo.nnz}\n")
        for i, j, v in zip(coo.row, coo.col, coo.data):
            fh.write(f"{i + 1} {j + 1} {float(v)!r}\n")

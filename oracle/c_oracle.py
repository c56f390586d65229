"""ctypes front end of oracle/c/cheb_oracle.c (CPU ORACLE: tests / CPU baseline only)."""

import ctypes
import os

import numpy as np

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "build", "liboracle.so")
_lib = None


def available():
    return os.path.exists(_LIB)


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(_LIB)
        p, i64, d, i = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        lib.oracle_cheb_moments.argtypes = [i64, p, p, p, d, d, i64, i, i64, p, p, i]
        lib.oracle_cheb_moments.restype = i
        lib.oracle_max_threads.restype = i
        lib.oracle_stencil_moments.argtypes = [i64, i64, i64, i, p, p, p, d, d, i64, i, i64, p, p, i]
        lib.oracle_stencil_moments.restype = i
        _lib = lib
    return _lib


def max_threads():
    return int(_load().oracle_max_threads())


def cheb_moments(csr, c, d, degree, probes, mode="doubling", threads=0):
    """Per-probe moments; probes is (n_vec, n) float64."""
    lib = _load()
    indptr = np.ascontiguousarray(csr.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
    data = np.ascontiguousarray(csr.data, dtype=np.float64)
    probes = np.ascontiguousarray(probes, dtype=np.float64)
    n_vec, n = probes.shape
    out = np.empty((n_vec, degree + 1))
    rc = lib.oracle_cheb_moments(n, indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, float(c), float(d),
                                 int(degree), 0 if mode == "direct" else 1, n_vec, probes.ctypes.data,
                                 out.ctypes.data, int(threads))
    if rc:
        raise RuntimeError(f"oracle_cheb_moments failed ({rc})")
    return out


def stencil_moments(op, c, d, degree, probes, mode="doubling", threads=0):
    """Per-probe moments of a periodic StencilOperator (no CSR is built)."""
    lib = _load()
    nx, ny, nz = op.shape
    offs = np.ascontiguousarray(np.asarray(op.offsets, dtype=np.int32).reshape(-1, 3))
    w = np.ascontiguousarray(op.weights, dtype=np.float64)
    diag = np.ascontiguousarray(op.diag, dtype=np.float64)
    probes = np.ascontiguousarray(probes, dtype=np.float64)
    n_vec, n = probes.shape
    out = np.empty((n_vec, degree + 1))
    rc = lib.oracle_stencil_moments(nx, ny, nz, len(w), offs.ctypes.data, w.ctypes.data, diag.ctypes.data, float(c),
                                    float(d), int(degree), 0 if mode == "direct" else 1, n_vec, probes.ctypes.data,
                                    out.ctypes.data, int(threads))
    if rc:
        raise RuntimeError(f"oracle_stencil_moments failed ({rc})")
    return out

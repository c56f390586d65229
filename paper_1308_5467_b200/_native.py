"""ctypes binding of ``libspecdens_b200.so`` (the C ABI in include/specdens_b200.h).

The shared library is built in-tree (``make -C paper_1308_5467_b200/csrc`` or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
every compute entry point raises, so a silent CPU path can never stand in for
the CUDA kernels.
"""

import ctypes
import os
import threading

from .errors import NumericalFailure

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspecdens_b200.so")

SDB_OK = 0
SDB_EINVAL = 1
SDB_ECUDA = 2
SDB_ENUMERIC = 3
SDB_ENOMEM = 4
SDB_EUNSUPPORTED = 5

SDB_CHEB_DIRECT = 0
SDB_CHEB_DOUBLING = 1
SDB_LEGENDRE = 2
SDB_DAMP_NONE = 0
SDB_DAMP_JACKSON = 1
SDB_REORTH = {"full": 0, "selective": 1, "none": 2}
SDB_LZ_OK = 0
SDB_LZ_BREAKDOWN = 1
SDB_LZ_NONFINITE = 2
SDB_LZ_ZERO_START = 3
SDB_FMT_CSR = 0
SDB_FMT_STENCIL = 1
SDB_MAX_BATCH = 256


class SdbMatrixInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("format", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("bytes", ctypes.c_int64),
    ]


class SdbStencilDesc(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int64),
        ("ny", ctypes.c_int64),
        ("nz", ctypes.c_int64),
        ("n_offsets", ctypes.c_int32),
        ("offsets", (ctypes.c_int32 * 3) * 26),
        ("weights", ctypes.c_double * 26),
        ("z_ghost", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_i = ctypes.c_int
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_d = ctypes.c_double
_p = ctypes.c_void_p
_sz = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/specdens_b200.h
SIGNATURES = {
    "sdb_last_error": (ctypes.c_char_p, []),
    "sdb_version": (_i, []),
    "sdb_block_ldv": (_i64, [_i64]),
    "sdb_matrix_create_csr": (_i, [_i, _i64, _i64, _p, _p, _i, _p, _p, ctypes.POINTER(_p)]),
    "sdb_matrix_create_stencil": (_i, [_i, ctypes.POINTER(SdbStencilDesc), _p, _p, ctypes.POINTER(_p)]),
    "sdb_matrix_get_info": (_i, [_p, ctypes.POINTER(SdbMatrixInfo)]),
    "sdb_matrix_band_info": (_i, [_p, ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "sdb_matrix_destroy": (None, [_p]),
    "sdb_pack_probes": (_i, [_p, _i64, _i64, _i64, _p, _p]),
    "sdb_unpack_block": (_i, [_p, _i64, _i64, _i64, _p, _p]),
    "sdb_unpack_signs": (_i, [_p, _i64, _i64, _i64, _p, _p]),
    "sdb_cheb_workspace_size": (_i, [_p, _i64, _i64, _i, ctypes.POINTER(_sz)]),
    "sdb_legendre_series": (_i, [_p, _i64, _p, _i64, _d, _p, _p, _p]),
    "sdb_haydock": (_i, [_p, _p, _p, _p, _i64, _i64, _p, _i64, _d, _p, _p, _p, _p]),
    "sdb_tridiag_resolvent": (_i, [_p, _p, _i64, _p, _i64, _p, _p, _p, _p, _p]),
    "sdb_dgl": (_i, [_p, _i64, _p, _i64, _d, _d, _d, _p, _p, _p, _p, _p, _p]),
    "sdb_mm_read": (_i, [ctypes.c_char_p, ctypes.POINTER(_p)]),
    "sdb_mm_info": (_i, [_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int32)]),
    "sdb_mm_export": (_i, [_p, _p, _p, _p]),
    "sdb_mm_free": (None, [_p]),
    "sdb_cheb_kernel": (ctypes.c_char_p, [_p, _i64, _i]),
    "sdb_cheb_moments": (_i, [_p, _d, _d, _i64, _i64, _i, _p, _p, _p, _sz, _p, ctypes.POINTER(ctypes.c_float)]),
    "sdb_cheb_partials_size": (_i, [_p, _i64, _i64, _i, ctypes.POINTER(_sz)]),
    "sdb_cheb_step": (_i, [_p, _d, _d, _i64, _i64, _i, _i64, _p, _p, _p, _p, _p, _sz, _p]),
    "sdb_cheb_step_halo": (_i, [_p, _d, _d, _i64, _i64, _i, _i64, _p, _p, _p, _p, _p, _sz, _p, _p, _p]),
    "sdb_zm_block_info": (_i, [_p, _i64, _i, ctypes.POINTER(_i64), ctypes.POINTER(_sz)]),
    "sdb_zm_pad_probes": (_i, [_p, _i64, _p, _p, _p]),
    "sdb_cheb_step_planes": (_i, [_p, _d, _d, _i64, _i64, _i, _i64, _i64, _i64, _p, _p, _p, _p, _p, _sz, _p]),
    "sdb_cheb_step_planes_halo": (_i, [_p, _d, _d, _i64, _i64, _i, _i64, _i64, _i64, _p, _p, _p, _p, _p, _sz, _p, _p,
                                       _p]),
    "sdb_cheb_reduce_planes": (_i, [_p, _i64, _i64, _i, _i64, _i64, _p, _p, _p]),
    "sdb_enable_peer_access": (_i, [_i, _i]),
    "sdb_cheb_reduce": (_i, [_p, _i64, _i64, _i, _p, _p, _p]),
    "sdb_moments_mean": (_i, [_p, _i64, _i64, _p, _p, _p]),
    "sdb_jackson_damping": (_i, [_i64, _p, _p]),
    "sdb_kpm_coefficients": (_i, [_p, _i64, _i64, _i, _p, _p]),
    "sdb_chebyshev_series": (_i, [_p, _i64, _p, _i64, _i, _d, _p, _p, _p]),
    "sdb_lanczos_workspace_size": (_i, [_p, _i64, _i64, ctypes.POINTER(_sz)]),
    "sdb_lanczos": (_i, [_p, _d, _d, _i64, _i64, _i, _p, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "sdb_ritz_quadrature": (_i, [_p, _p, _p, _i64, _i64, _p, _p, _p]),
    "sdb_ritz_residual_bounds": (_i, [_p, _p, _p, _i64, _i64, _p, _p, _p]),
    "sdb_pool_nodes": (_i, [_p, _p, _p, _i64, _i64, _d, _p, _p, ctypes.POINTER(_i64), _p]),
    "sdb_blur_nodes": (_i, [_p, _p, _i64, _d, _i, _d, _p, _i64, _p, _p]),
    "sdb_cdos_refine": (_i, [_p, _p, _i64, _d, _d, _d, _p, _i64, _p, _p, _p, _p, _p, _p, ctypes.POINTER(_i64), _p]),
}

_lock = threading.Lock()
_lib = None


class NativeLibraryMissing(ImportError):
    pass


def load():
    """Load (once) and return the native library; raise if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_1308_5467_b200/csrc` (there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error():
    msg = load().sdb_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc, what=""):
    """Map a C-ABI status code to the reference's exception types."""
    if rc == SDB_OK:
        return
    msg = last_error() or what
    if rc == SDB_EINVAL:
        raise ValueError(msg)
    if rc == SDB_ENUMERIC:
        raise NumericalFailure(msg)
    if rc == SDB_ENOMEM:
        raise MemoryError(msg)
    if rc == SDB_EUNSUPPORTED:
        raise TypeError(msg)
    raise RuntimeError(msg)


def call(name, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc

"""Device plumbing between the reference-shaped API and the C ABI.

PyTorch is used only for device memory, pinned host buffers and streams; all
arithmetic on the hot path runs in the kernels of ``libspecdens_b200.so``.
"""

import ctypes
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import NumericalFailure
from .operators import device_matrix, resolve
from .stochastic import draw_block

SPECTRUM_ESCAPE_HINT = (
    "the recurrence produced non-finite moments, which usually means the "
    "spectrum escapes the mapped interval [-1, 1]; widen the spectral "
    "interval (larger safety margin or more Lanczos steps for the bounds)"
)


def _torch():
    import torch

    return torch


def is_device_list(device):
    """``device`` may be one CUDA device index or a sequence of them (probe sharding)."""
    return isinstance(device, (list, tuple))


def require_cuda(device=None):
    """The CUDA device to compute on (for a device list: its first entry,
    where the sharded per-probe rows are gathered and evaluated)."""
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1308_5467_b200 needs a CUDA device (sm_100a); no GPU is visible and there is no CPU fallback"
        )
    _native.load()
    if is_device_list(device):
        if not device:
            raise ValueError("empty device list")
        device = device[0]
    if device is None:
        device = torch.cuda.current_device()
    return int(device)


def stream_ptr(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def block_ldv(n_vec):
    v = _native.load().sdb_block_ldv(int(n_vec))
    if v < 0:
        raise ValueError(f"probe batch size {n_vec} outside [1, {_native.SDB_MAX_BATCH}]")
    return int(v)


def batches(n_vec, batch=_native.SDB_MAX_BATCH):
    """Contiguous probe ranges of at most ``batch`` probes."""
    import os

    if os.environ.get("SDB_BATCH"):
        batch = max(1, min(batch, int(os.environ["SDB_BATCH"])))
    return [(s, min(batch, n_vec - s)) for s in range(0, n_vec, batch)]


@dataclass
class Staged:
    """A probe batch resident on the device as an n x ldv block."""

    block: object   # torch float64 (n, ldv)
    ldv: int
    h2d_bytes: int


def stage_probes(source, start, count, n, device, stream):
    """Draw probes start..start+count-1 on the host and pack them on device."""
    torch = _torch()
    if int(source.dim) != n:
        raise ValueError(f"probe dimension {source.dim} does not match operator dimension {n}")
    ldv = block_ldv(count)
    if getattr(source, "kind", None) == "rademacher" and hasattr(source, "draw_block_signs"):
        bits = source.draw_block_signs(start, count)
        dev_b = torch.empty(bits.shape, dtype=torch.uint8, device=device)
        dev_b.copy_(bits, non_blocking=True)
        block = torch.empty((n, ldv), dtype=torch.float64, device=device)
        _native.call("sdb_unpack_signs", ptr(dev_b), count, n, ldv, ptr(block), stream)
        block._sdb_keepalive = (bits, dev_b)
        return Staged(block=block, ldv=ldv, h2d_bytes=int(bits.numel()))
    host = draw_block(source, start, count)
    if not isinstance(host, torch.Tensor):
        host = torch.from_numpy(np.ascontiguousarray(host, dtype=np.float64))
    dev_t = torch.empty((count, n), dtype=torch.float64, device=device)
    dev_t.copy_(host, non_blocking=True)
    block = torch.empty((n, ldv), dtype=torch.float64, device=device)
    _native.call("sdb_pack_probes", ptr(dev_t), count, n, ldv, ptr(block), stream)
    # keep the host buffer alive until the stream has consumed it
    block._sdb_keepalive = (host, dev_t)
    return Staged(block=block, ldv=ldv, h2d_bytes=8 * count * n)


def pack_device_probes(probes_t, device, stream):
    """Pack an on-device (count, n) probe tensor into an n x ldv block."""
    torch = _torch()
    count, n = probes_t.shape
    ldv = block_ldv(count)
    block = torch.empty((n, ldv), dtype=torch.float64, device=device)
    _native.call("sdb_pack_probes", ptr(probes_t), count, n, ldv, ptr(block), stream)
    return Staged(block=block, ldv=ldv, h2d_bytes=0)


class Workspace:
    """Grow-only device scratch buffers, one per (device, stream).

    Work on a stream is ordered, so successive calls on the same stream may
    share a buffer; calls on different streams (other host threads, the
    shards of a multi-device estimate) each get their own and cannot race.
    """

    _lock = threading.Lock()
    _buffers = {}

    @classmethod
    def get(cls, device, nbytes):
        torch = _torch()
        key = (int(device), int(torch.cuda.current_stream(device).cuda_stream))
        with cls._lock:
            buf = cls._buffers.get(key)
            if buf is None or buf.numel() < nbytes:
                cls._buffers.pop(key, None)
                buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
                cls._buffers[key] = buf
        return buf

    @classmethod
    def release(cls, device=None, stream=None):
        """Drop the buffers (all, or those of one device / one stream)."""
        with cls._lock:
            for key in list(cls._buffers):
                if (device is None or key[0] == int(device)) and (stream is None or key[1] == int(stream)):
                    del cls._buffers[key]


# ---------------------------------------------------------------------------
# KPM moments


@dataclass
class MomentRun:
    zeta_pp: object        # torch (n_vec, degree+1) on device
    n: int
    resolved: object
    matvecs_per_probe: int
    step_ms: float         # CUDA-event time of the recurrence kernels
    h2d_bytes: int
    dm: object


# ---------------------------------------------------------------------------
# probe sharding over several devices of one process (probe
# recurrences are independent units)


def shard_range(n_vec, world, rank):
    """Contiguous probe range of shard ``rank``: sizes differ by at most one."""
    base, extra = divmod(n_vec, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


class ShiftedSource:
    """Probe i of this view is probe start+i of the underlying source."""

    def __init__(self, src, start):
        self.src, self.start, self.dim = src, start, src.dim
        self.kind = getattr(src, "kind", None)
        if hasattr(src, "draw_block_signs"):
            self.draw_block_signs = lambda s, c: src.draw_block_signs(self.start + s, c)

    def draw(self, i):
        return self.src.draw(self.start + i)

    def draw_block(self, start, count):
        return draw_block(self.src, self.start + start, count)


def run_sharded(fn, n_vec, devices, source=None, probes=None):
    """Run ``fn(shard_source, shard_probes, count, device)`` for every shard.

    Shard r is the contiguous probe range ``shard_range(n_vec, len(devices),
    r)`` on ``devices[r]`` (a device may appear several times), each on its
    own host thread and CUDA stream, so the shards of one device queue behind
    each other while different devices run concurrently.  Returns the shard
    results in probe order; every shard's stream has been synchronised.
    """
    torch = _torch()
    devices = [int(d) for d in devices][:max(1, n_vec)]
    world = len(devices)

    def work(r):
        start, count = shard_range(n_vec, world, r)
        d = devices[r]
        with torch.cuda.device(d):
            stream = torch.cuda.Stream(device=d)
            with torch.cuda.stream(stream):
                src = ShiftedSource(source, start) if source is not None else None
                pr = None
                if probes is not None:
                    pr = probes[start:start + count]
                    if pr.device.index != d:
                        pr = pr.to(d)
                out = fn(src, pr, count, d)
            stream.synchronize()
            Workspace.release(d, stream.cuda_stream)
        return out

    if world == 1:
        return [work(0)]
    with ThreadPoolExecutor(max_workers=world) as ex:
        return list(ex.map(work, range(world)))


def run_chebyshev(op, degree, source, n_vec, mode, device=None, probes=None, time_steps=False):
    """Per-probe Chebyshev moments of the resolved operator.

    ``device``: one CUDA device, or a list of devices: the probes are then
    sharded over them (one contiguous range per list entry, one stream each)
    and the per-probe rows gathered on the first device, in probe order.
    ``probes`` optionally supplies an on-device (n_vec, n) tensor instead of
    drawing from ``source`` (used by the benchmark's device-resident leg and
    the multi-GPU shard, which pass their own slice).
    """
    torch = _torch()
    if is_device_list(device):
        primary = require_cuda(device)
        res = resolve(op)
        for d in sorted(set(int(x) for x in device)):  # one upload per device, before the shards start
            with torch.cuda.device(d):
                device_matrix(res.base, d, stream_ptr(d))
                torch.cuda.current_stream(d).synchronize()
        runs = run_sharded(lambda src, pr, count, d: run_chebyshev(op, degree, src, count, mode, device=d, probes=pr,
                                                                   time_steps=time_steps),
                           n_vec, device, source=source if probes is None else None, probes=probes)
        with torch.cuda.device(primary):
            zeta_pp = torch.cat([r.zeta_pp.to(primary) for r in runs], dim=0)
        return MomentRun(zeta_pp=zeta_pp, n=runs[0].n, resolved=runs[0].resolved,
                         matvecs_per_probe=runs[0].matvecs_per_probe, step_ms=max(r.step_ms for r in runs),
                         h2d_bytes=sum(r.h2d_bytes for r in runs), dm=runs[0].dm)
    device = require_cuda(device)
    res = resolve(op)
    n = res.dim
    if res.d == 0.0:
        raise ValueError("spectral halfwidth must be non-zero")
    with torch.cuda.device(device):
        stream = stream_ptr(device)
        dm = device_matrix(res.base, device, stream)
        zeta_pp = torch.empty((n_vec, degree + 1), dtype=torch.float64, device=device)
        lib = _native.load()
        step_ms_total = 0.0
        h2d = 0
        for start, count in batches(n_vec):
            if probes is not None:
                staged = pack_device_probes(probes[start:start + count], device, stream)
            else:
                staged = stage_probes(source, start, count, n, device, stream)
            h2d += staged.h2d_bytes
            need = ctypes.c_size_t()
            _native.check(lib.sdb_cheb_workspace_size(dm.handle, count, degree, mode, ctypes.byref(need)))
            ws = Workspace.get(device, need.value)
            out = zeta_pp[start:start + count]
            ms = ctypes.c_float(0.0)
            _native.check(lib.sdb_cheb_moments(dm.handle, res.c, res.d, count, degree, mode, ptr(staged.block),
                                               ptr(out), ptr(ws), ws.numel(), stream,
                                               ctypes.byref(ms) if time_steps else None))
            step_ms_total += ms.value
        per_probe = (degree + 1) // 2 if mode == _native.SDB_CHEB_DOUBLING else degree
    return MomentRun(zeta_pp=zeta_pp, n=n, resolved=res, matvecs_per_probe=per_probe, step_ms=step_ms_total,
                     h2d_bytes=h2d, dm=dm)


def credit_counters(resolved, n_vec, per_probe):
    for c in resolved.counters:
        c.count += n_vec * per_probe


def mean_moments(zeta_pp, device):
    """Probe-ordered mean (kpm.py:135) on device; returns (zeta_dev, flag_dev)."""
    torch = _torch()
    n_vec, m1 = zeta_pp.shape
    zeta = torch.empty(m1, dtype=torch.float64, device=device)
    flag = torch.zeros(1, dtype=torch.int32, device=device)
    _native.call("sdb_moments_mean", ptr(zeta_pp), n_vec, m1 - 1, ptr(zeta), ptr(flag), stream_ptr(device))
    return zeta, flag


def kpm_density_device(zeta_dev, degree, n, damping, t_dev, d, device):
    """mu = coefficients(zeta), values = Clenshaw(mu, t)/sqrt(1-t^2), density = values/d."""
    torch = _torch()
    stream = stream_ptr(device)
    mu = torch.empty(degree + 1, dtype=torch.float64, device=device)
    _native.call("sdb_kpm_coefficients", ptr(zeta_dev), degree, n, damping, ptr(mu), stream)
    n_pts = t_dev.numel()
    values = torch.empty(n_pts, dtype=torch.float64, device=device)
    density = torch.empty(n_pts, dtype=torch.float64, device=device)
    _native.call("sdb_chebyshev_series", ptr(mu), degree, ptr(t_dev), n_pts, 1, float(d), ptr(values),
                 ptr(density), stream)
    return mu, values, density


def to_device(arr, device):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64)).to(device, non_blocking=False)


class Timer:
    def __init__(self):
        self.t0 = time.perf_counter()

    def elapsed(self):
        return time.perf_counter() - self.t0

"""Probe vectors (mirror of specdens/stochastic.py:20-74) and their staging.

``ProbeVectorSource`` keeps the reference's contract exactly: probe ``index``
is drawn from ``Philox(SeedSequence(seed, spawn_key=(stream, index)))``
(stochastic.py:40-54), so the same (kind, seed, dim, stream, index) gives the
same vector as the reference in the same NumPy.  NumPy's generator streams
carry no cross-version guarantee, so probes are always drawn on the host with
the NumPy of this process and uploaded ("the same injected probe vectors").

The engine accepts any object with ``draw(index)`` and ``dim``.  Sources of
this class additionally keep the most recently drawn block in pinned host
memory (``draw_block``): draws are pure functions of the index, so re-using
them is unobservable, and repeated estimates over the same probes then cost
one host->device copy instead of a re-draw.
"""

import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

PROBE_KINDS = ("gaussian", "rademacher", "basis")
INTERVAL_STREAM = 0xB0

# pinned-memory budget for the per-source block cache
PINNED_CACHE_BYTES = 8 << 30


@dataclass(frozen=True)
class ProbeVectorSource:
    kind: str
    seed: int
    dim: int
    stream: int = 0
    # drawn blocks kept in pinned host memory (a pure-function cache: the value
    # object stays immutable for every observer); guarded by _lock
    _cache: dict = field(default_factory=dict, compare=False, repr=False, hash=False)
    _lock: object = field(default_factory=threading.Lock, compare=False, repr=False, hash=False)

    def __post_init__(self):
        if self.kind not in PROBE_KINDS:
            raise ValueError(f"unknown probe kind {self.kind!r}, expected one of {PROBE_KINDS}")
        if self.dim < 1:
            raise ValueError("probe dimension must be positive")

    def draw(self, index):
        """Probe vector ``index`` (deterministic in (seed, stream, index))."""
        if self.kind == "basis":
            if not 0 <= index < self.dim:
                raise ValueError(f"basis probe index {index} out of range for dimension {self.dim}")
            v = np.zeros(self.dim)
            v[index] = np.sqrt(self.dim)
            return v
        ss = np.random.SeedSequence(self.seed, spawn_key=(self.stream, index))
        rng = np.random.Generator(np.random.Philox(ss))
        if self.kind == "gaussian":
            return rng.standard_normal(self.dim)
        return rng.integers(0, 2, self.dim) * 2.0 - 1.0

    @property
    def is_exhaustive(self):
        return self.kind == "basis"

    def with_stream(self, stream):
        return ProbeVectorSource(self.kind, self.seed, self.dim, stream)

    def draw_block_signs(self, start, count):
        """Rademacher probes start..start+count-1 as packed sign bits.

        (count, ceil(dim/8)) uint8, bit i of row l set iff probe entry i is
        +1 (NumPy packbits, little bit order).  The +-1 values are exact, so
        this is the same input in 1/64 of the bytes; cached like draw_block.
        """
        if self.kind != "rademacher":
            raise ValueError("sign packing applies to rademacher probes only")
        import torch

        key = ("signs", start, count)
        with self._lock:
            hit = self._cache.get(key)
        if hit is not None:
            return hit
        nb = (int(self.dim) + 7) // 8
        out = torch.empty((count, nb), dtype=torch.uint8, pin_memory=torch.cuda.is_available())
        arr = out.numpy()

        def one(i):
            ss = np.random.SeedSequence(self.seed, spawn_key=(self.stream, start + i))
            rng = np.random.Generator(np.random.Philox(ss))
            arr[i] = np.packbits(rng.integers(0, 2, self.dim).astype(np.uint8), bitorder="little")

        if count >= 4:
            with ThreadPoolExecutor(max_workers=min(_DRAW_THREADS, count)) as ex:
                list(ex.map(one, range(count)))
        else:
            for i in range(count):
                one(i)
        _cache_put(self._cache, self._lock, key, out)
        return out

    def draw_block(self, start, count, out=None):
        """Probes start..start+count-1 as a (count, dim) float64 array.

        Uses a one-entry cache of pinned host memory (see module doc).
        """
        return _draw_block(self, start, count, out, cache=self._cache, lock=self._lock)


_pool_lock = threading.Lock()
# host threads that draw probe rows in parallel (NumPy's generators release the GIL)
_DRAW_THREADS = max(1, min(32, os.cpu_count() or 8))


def _draw_rows(source, start, count, out):
    def one(i):
        out[i] = source.draw(start + i)

    if count >= 4:
        # drawing is NumPy C code that releases the GIL; fill rows in parallel
        with ThreadPoolExecutor(max_workers=min(_DRAW_THREADS, count)) as ex:
            list(ex.map(one, range(count)))
    else:
        for i in range(count):
            one(i)


def _cache_put(cache, lock, key, block):
    """Insert a drawn block; the oldest blocks go once the pinned budget is exceeded."""
    with lock:
        cache.pop(key, None)
        cache[key] = block
        total = sum(b.numel() * b.element_size() for b in cache.values())
        for k in list(cache):
            if total <= PINNED_CACHE_BYTES or k == key:
                break
            b = cache.pop(k)
            total -= b.numel() * b.element_size()


def _draw_block(source, start, count, out, cache=None, lock=None):
    import torch

    key = ("values", start, count)
    if cache is not None:
        with lock:
            hit = cache.get(key)
        if hit is not None:
            if out is not None:
                out.copy_(hit)
                return out
            return hit
    nbytes = 8 * count * int(source.dim)
    if out is None:
        pin = torch.cuda.is_available() and (cache is None or nbytes <= PINNED_CACHE_BYTES)
        out = torch.empty((count, int(source.dim)), dtype=torch.float64, pin_memory=pin)
    _draw_rows(source, start, count, out.numpy())
    if cache is not None and nbytes <= PINNED_CACHE_BYTES:
        _cache_put(cache, lock, key, out)
    return out


def draw_block(source, start, count):
    """(count, dim) host tensor of probes from any source with ``draw``."""
    if hasattr(source, "draw_block"):
        return source.draw_block(start, count)
    return _draw_block(source, start, count, None, cache=None)


def map_probes(fn, n_vec, threads=None):
    """Apply ``fn`` to 0..n_vec-1 in index order (stochastic.py:64-74)."""
    indices = range(n_vec)
    if threads is not None and threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            return list(ex.map(fn, indices))
    return [fn(i) for i in indices]

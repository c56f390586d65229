"""Row-partitioned KPM moments for periodic stencils.

The grid's z-planes are split into contiguous slabs, one per rank (GPU).
Each slab keeps, in every n x ldv block it holds, one ghost plane below and
one above its own planes.  Per recurrence step:

  1. every slab runs the fused step kernel on its own rows (``sdb_cheb_step``
     with a z-ghost stencil handle: z is not wrapped, the neighbours of the
     first / last own plane are read from the ghost planes);
  2. halo exchange: a slab's first own plane of w_{k+1} becomes the upper
     ghost of the slab below it, its last own plane the lower ghost of the
     slab above it (periodic in z) -- a device copy when both slabs live in
     this process, an NCCL send/recv pair otherwise (2 x nx*ny*ldv*8 bytes
     received per slab per step: 33.6 MB at 256^3 with 32 probes).

With an exchange between ranks (NCCL) the step is split so the transfer
overlaps the bulk of the SpMM: the slab's first and last own planes are
computed first (two single-plane z-ghost handles on the same block memory),
the halo send/recv of those planes is issued on a communication stream, and
the interior planes are computed on the compute stream meanwhile.  The next
step's boundary planes wait for the exchange; its interior does not need it.

Moments are sums over rows, so each slab reduces its own partials into
per-probe moments and one all-reduce over ranks at the end gives the global
per-probe moments (the doubling transform is linear, so it commutes with the
sum).  The step's compute and the driver's exchange are passed in as
callables so the same driver runs the CUDA path (``DeviceSlab``) and a CPU
reference slab in the multi-process gloo tests.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from . import engine as E
from .distributed import shard_range
from .operators import SlabStencil, StencilOperator, device_matrix


@dataclass
class SlabPlan:
    """Which planes each slab owns."""

    nz: int
    n_slabs: int

    def planes(self, s):
        return shard_range(self.nz, self.n_slabs, s)  # (z0, count)

    def neighbours(self, s):
        return (s - 1) % self.n_slabs, (s + 1) % self.n_slabs


def halo_exchange(slabs, plan, blocks, group=None, rank_of_slab=None):
    """Refresh the ghost planes of ``blocks[s]`` for every local slab s.

    ``slabs``: local slab indices; ``blocks[s]``: tensor view (nzl+2, nxy, ldv)
    of slab s's current w block (ghost planes at [0] and [-1]).
    ``rank_of_slab``: maps a slab to its rank (None -> all slabs local).
    """
    import torch.distributed as dist

    local = set(slabs)
    ops = []
    for s in slabs:
        lo, hi = plan.neighbours(s)
        blk = blocks[s]
        # ghost below = last own plane of slab lo; ghost above = first own plane of slab hi
        if lo in local:
            blk[0].copy_(blocks[lo][-2])
        if hi in local:
            blk[-1].copy_(blocks[hi][1])
    if rank_of_slab is None:
        return
    for s in slabs:  # sends first, then receives (matching order for any world size)
        lo, hi = plan.neighbours(s)
        blk = blocks[s]
        if lo not in local:
            ops.append(dist.P2POp(dist.isend, blk[1].contiguous() if not blk[1].is_contiguous() else blk[1],
                                  rank_of_slab(lo), group))
        if hi not in local:
            ops.append(dist.P2POp(dist.isend, blk[-2], rank_of_slab(hi), group))
    for s in slabs:
        lo, hi = plan.neighbours(s)
        blk = blocks[s]
        if hi not in local:
            ops.append(dist.P2POp(dist.irecv, blk[-1], rank_of_slab(hi), group))
        if lo not in local:
            ops.append(dist.P2POp(dist.irecv, blk[0], rank_of_slab(lo), group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def ghosted_probe_block(source, start, count, parent_shape, z0, nzl, ldv, out):
    """Fill ``out`` (nzl+2, nxy, ldv) with planes z0-1 .. z0+nzl (periodic) of
    probes start..start+count-1, padding columns zero."""
    nx, ny, nz = parent_shape
    nxy = nx * ny
    planes = [(z0 - 1) % nz] + list(range(z0, z0 + nzl)) + [(z0 + nzl) % nz]
    host = np.zeros((nzl + 2, nxy, ldv))
    for l in range(count):
        v = np.asarray(source.draw(start + l)).reshape(nz, nxy)
        host[:, :, l] = v[planes]
    out.copy_(__import__("torch").from_numpy(host))


class DeviceSlab:
    """One slab on one GPU: z-ghost stencil handle + ghosted blocks."""

    def __init__(self, op, plan, s, n_vec, degree, mode, device):
        import torch

        self.s = s
        self.z0, self.nzl = plan.planes(s)
        self.slab = SlabStencil(op, self.z0, self.z0 + self.nzl)
        self.device = device
        with torch.cuda.device(device):
            self.torch_stream = torch.cuda.current_stream(device)
        self.stream = ctypes.c_void_p(self.torch_stream.cuda_stream)
        self.dm = device_matrix(self.slab, device, self.stream)
        self.ldv = E.block_ldv(n_vec)
        nx, ny, _ = op.shape
        self.nxy = nx * ny
        shape = (self.nzl + 2, self.nxy, self.ldv)
        self.blocks = [torch.zeros(shape, dtype=torch.float64, device=device) for _ in range(3)]
        need = __import__("ctypes").c_size_t()
        _native.check(_native.load().sdb_cheb_partials_size(self.dm.handle, n_vec, degree, mode,
                                                            __import__("ctypes").byref(need)))
        self.partials = torch.empty(max(need.value, 8) // 8 + 1, dtype=torch.float64, device=device)
        self.n_vec, self.degree, self.mode = n_vec, degree, mode
        # boundary / interior split (overlapped exchange): single-plane handles
        # for the first and last own plane, one for the planes between them;
        # each part owns a partials buffer, its moments are summed in reduce()
        self.parts = {}
        if self.nzl >= 3:
            spans = {"lo": (0, 1), "int": (1, self.nzl - 1), "hi": (self.nzl - 1, self.nzl)}
            for name, (a, b) in spans.items():
                sub = SlabStencil(op, self.z0 + a, self.z0 + b)
                dm = device_matrix(sub, device, self.stream)
                _native.check(_native.load().sdb_cheb_partials_size(dm.handle, n_vec, degree, mode,
                                                                    ctypes.byref(need)))
                part = torch.empty(max(need.value, 8) // 8 + 1, dtype=torch.float64, device=device)
                self.parts[name] = (sub, dm, a, part)
        self.split_used = False

    def own(self, t):
        """Pointer to the first own row of a ghosted block."""
        return E.ptr(t[1])

    def step(self, k, c, d, cur, prev, nxt, v0):
        _native.call("sdb_cheb_step", self.dm.handle, c, d, self.n_vec, self.degree, self.mode, k, self.own(cur),
                     self.own(prev) if prev is not None else None, self.own(nxt), self.own(v0),
                     E.ptr(self.partials), self.partials.numel() * 8, self.stream)

    def step_halo(self, k, c, d, cur, prev, nxt, v0, halo_lo, halo_hi):
        """Step whose kernel epilogue also stores the first / last own plane of
        w_{k+1} into the neighbours' ghost planes (tensors on this or a peer
        device) -- the fused compute + halo exchange."""
        _native.call("sdb_cheb_step_halo", self.dm.handle, c, d, self.n_vec, self.degree, self.mode, k,
                     self.own(cur), self.own(prev) if prev is not None else None, self.own(nxt), self.own(v0),
                     E.ptr(self.partials), self.partials.numel() * 8, E.ptr(halo_lo), E.ptr(halo_hi), self.stream)

    def step_part(self, name, k, c, d, cur, prev, nxt, v0):
        """Step of one part ('lo', 'int', 'hi') of the slab's own planes: the
        part's handle reads its z neighbours from the adjacent planes of the
        same ghosted block (own planes, or the slab's ghost planes at the ends)."""
        _, dm, a, part = self.parts[name]
        row = lambda t: E.ptr(t[1 + a])  # noqa: E731
        _native.call("sdb_cheb_step", dm.handle, c, d, self.n_vec, self.degree, self.mode, k, row(cur),
                     row(prev) if prev is not None else None, row(nxt), row(v0), E.ptr(part), part.numel() * 8,
                     self.stream)
        self.split_used = True

    def reduce(self):
        import torch

        if self.split_used:
            total = None
            for _, dm, _, part in self.parts.values():
                z = torch.empty((self.n_vec, self.degree + 1), dtype=torch.float64, device=self.device)
                _native.call("sdb_cheb_reduce", dm.handle, self.n_vec, self.degree, self.mode, E.ptr(part),
                             E.ptr(z), self.stream)
                total = z if total is None else total + z
            return total
        zeta_pp = torch.empty((self.n_vec, self.degree + 1), dtype=torch.float64, device=self.device)
        _native.call("sdb_cheb_reduce", self.dm.handle, self.n_vec, self.degree, self.mode, E.ptr(self.partials),
                     E.ptr(zeta_pp), self.stream)
        return zeta_pp


class PlaneSlab:
    """One slab on one GPU in the z-march layout (periodic 7/27-point grids):
    full-size ghost-padded blocks [nz][ny+2][nx+2][ldv] of the whole grid, of
    which this slab computes its own planes [z0, z0+nzl) with the TMA z-march
    kernel restricted to that range (``sdb_cheb_step_planes``) and holds valid
    data only there plus the two neighbour planes the exchange fills.  The
    unused planes cost memory only (3 x 4.4 GB at 256^3 x 32 probes, of 180 GB).

    Parts: first own plane, interior, last own plane (``step_part``), so the
    boundary planes can be exchanged while the interior is computed."""

    def __init__(self, op, plan, s, n_vec, degree, mode, device, info=None):
        import torch

        self.s = s
        self.z0, self.nzl = plan.planes(s)
        self.nz = op.shape[2]
        self.device = device
        with torch.cuda.device(device):
            self.torch_stream = torch.cuda.current_stream(device)
        self.stream = ctypes.c_void_p(self.torch_stream.cuda_stream)
        self.dm = device_matrix(op, device, self.stream)
        pd, bb = info if info is not None else plane_layout(self.dm, n_vec, mode)
        if pd == 0:
            raise TypeError("the z-march layout does not apply to this operator")
        self.plane_doubles = pd
        self.n_vec, self.degree, self.mode = n_vec, degree, mode
        self.ldv = E.block_ldv(n_vec)
        flat = [torch.empty(bb // 8, dtype=torch.float64, device=device) for _ in range(3)]
        for f in flat[1:]:
            f.fill_(float("nan"))  # planes the exchange does not fill must never be read
        self.blocks = [f[:self.nz * pd].view(self.nz, pd) for f in flat]
        z0, z1 = self.z0, self.z0 + self.nzl
        if self.nzl >= 3:
            self.parts = {"lo": (z0, z0 + 1), "int": (z0 + 1, z1 - 1), "hi": (z1 - 1, z1)}
        else:
            self.parts = {}
        need = ctypes.c_size_t()
        _native.check(_native.load().sdb_cheb_partials_size(self.dm.handle, n_vec, degree, mode, ctypes.byref(need)))
        self.partials = {name: torch.empty(max(need.value, 8) // 8 + 1, dtype=torch.float64, device=device)
                         for name in list(self.parts) + ["all"]}  # one partials buffer per plane range
        self.used = set()

    def stage_probes(self, source):
        """Probes 0..n_vec-1 (drawn on the host as the reference does) -> padded block 0."""
        staged = E.stage_probes(source, 0, self.n_vec, int(source.dim), self.device, self.stream)
        _native.call("sdb_zm_pad_probes", self.dm.handle, self.n_vec, E.ptr(staged.block), E.ptr(self.blocks[0]),
                     self.stream)
        self._keep = staged

    def _step(self, name, z_lo, z_hi, k, c, d, cur, prev, nxt, v0):
        part = self.partials[name]
        _native.call("sdb_cheb_step_planes", self.dm.handle, c, d, self.n_vec, self.degree, self.mode, k, z_lo, z_hi,
                     E.ptr(cur), E.ptr(prev) if prev is not None else None, E.ptr(nxt), E.ptr(v0), E.ptr(part),
                     part.numel() * 8, self.stream)
        self.used.add((name, z_lo, z_hi))

    def step(self, k, c, d, cur, prev, nxt, v0):
        self._step("all", self.z0, self.z0 + self.nzl, k, c, d, cur, prev, nxt, v0)

    def step_part(self, name, k, c, d, cur, prev, nxt, v0):
        z_lo, z_hi = self.parts[name]
        self._step(name, z_lo, z_hi, k, c, d, cur, prev, nxt, v0)

    def step_halo(self, k, c, d, cur, prev, nxt, v0, halo_lo, halo_hi):
        """Step of the slab's planes whose z-march epilogue also stores its
        first / last plane of w_{k+1} into the neighbours' full-size blocks
        (``halo_lo`` / ``halo_hi``: tensors on this or a peer device, or None)."""
        part = self.partials["all"]
        z0, z1 = self.z0, self.z0 + self.nzl
        _native.call("sdb_cheb_step_planes_halo", self.dm.handle, c, d, self.n_vec, self.degree, self.mode, k, z0,
                     z1, E.ptr(cur), E.ptr(prev) if prev is not None else None, E.ptr(nxt), E.ptr(v0), E.ptr(part),
                     part.numel() * 8, E.ptr(halo_lo) if halo_lo is not None else None,
                     E.ptr(halo_hi) if halo_hi is not None else None, self.stream)
        self.used.add(("all", z0, z1))

    def reduce(self):
        import torch

        total = None
        for name, z_lo, z_hi in sorted(self.used):
            z = torch.empty((self.n_vec, self.degree + 1), dtype=torch.float64, device=self.device)
            _native.call("sdb_cheb_reduce_planes", self.dm.handle, self.n_vec, self.degree, self.mode, z_lo, z_hi,
                         E.ptr(self.partials[name]), E.ptr(z), self.stream)
            total = z if total is None else total + z
        return total


def plane_layout(dm, n_vec, mode):
    """(doubles per padded plane, bytes per padded block); (0, 0) when the
    z-march layout does not apply (non-grid stencil, CSR, odd shapes)."""
    pd, bb = ctypes.c_int64(), ctypes.c_size_t()
    _native.check(_native.load().sdb_zm_block_info(dm.handle, n_vec, mode, ctypes.byref(pd), ctypes.byref(bb)))
    return pd.value, bb.value


def plane_exchange(slabs, plan, blocks, group=None, rank_of_slab=None):
    """Halo exchange on full-size blocks: slab s receives plane z0-1 from its
    lower neighbour and plane z0+nzl from its upper neighbour (periodic), each
    stored at the same global plane index; local slabs copy, remote slabs use
    NCCL send/recv (sends first, lower then upper; receives upper then lower,
    so any world size, including 2, matches)."""
    import torch.distributed as dist

    by_s = {sl.s: sl for sl in slabs}
    nz = plan.nz
    for sl in slabs:
        lo, hi = plan.neighbours(sl.s)
        below, above = (sl.z0 - 1) % nz, (sl.z0 + sl.nzl) % nz
        if lo in by_s and lo != sl.s:
            blocks[sl.s][below].copy_(blocks[lo][below])
        if hi in by_s and hi != sl.s:
            blocks[sl.s][above].copy_(blocks[hi][above])
    if rank_of_slab is None:
        return
    ops = []
    for sl in slabs:
        lo, hi = plan.neighbours(sl.s)
        if lo not in by_s:
            ops.append(dist.P2POp(dist.isend, blocks[sl.s][sl.z0], rank_of_slab(lo), group))
        if hi not in by_s:
            ops.append(dist.P2POp(dist.isend, blocks[sl.s][sl.z0 + sl.nzl - 1], rank_of_slab(hi), group))
    for sl in slabs:
        lo, hi = plan.neighbours(sl.s)
        if hi not in by_s:
            ops.append(dist.P2POp(dist.irecv, blocks[sl.s][(sl.z0 + sl.nzl) % nz], rank_of_slab(hi), group))
        if lo not in by_s:
            ops.append(dist.P2POp(dist.irecv, blocks[sl.s][(sl.z0 - 1) % nz], rank_of_slab(lo), group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def run_rowpartition_p2p(slabs, plan, c, d, degree, mode):
    """All slabs in this process (one or several devices): every step kernel
    pushes its boundary planes straight into the neighbours' ghost planes (no
    separate exchange, no NCCL).  Step k+1 of a slab waits for its two
    neighbours' step k (stream order on one device, CUDA events across
    devices): their pushes have landed in its ghosts and they are done reading
    the ghosts it is about to overwrite."""
    import torch

    steps = (degree + 1) // 2 if mode == _native.SDB_CHEB_DOUBLING else degree
    by_id = {sl.s: sl for sl in slabs}
    if set(by_id) != set(range(plan.n_slabs)):
        raise ValueError("the p2p exchange needs every slab in this process")
    devices = sorted({sl.device for sl in slabs})
    for a in devices:
        for b in devices:
            _native.call("sdb_enable_peer_access", a, b)
    multi = len(devices) > 1
    full = hasattr(slabs[0], "plane_doubles")
    for sl in slabs:
        if full:
            sl.used.clear()
    cur = {s: by_id[s].blocks[0] for s in by_id}
    prev = {s: None for s in by_id}
    done = {}
    for k in range(max(steps, 1)):
        nxt = {s: by_id[s].blocks[1] if k == 0 else (by_id[s].blocks[2] if k == 1 else prev[s]) for s in by_id}
        push = steps > 0 and k + 1 < steps
        events = {}
        for s, sl in by_id.items():
            lo, hi = plan.neighbours(s)
            if multi and k > 0:
                for nb in {lo, hi}:
                    sl.torch_stream.wait_event(done[nb])
            if push and full:  # neighbours' full-size blocks, same global plane index
                sl.step_halo(k, c, d, cur[s], prev[s], nxt[s], sl.blocks[0], nxt[lo] if lo != s else None,
                             nxt[hi] if hi != s else None)
            elif push:  # neighbours' ghost planes
                sl.step_halo(k, c, d, cur[s], prev[s], nxt[s], sl.blocks[0], nxt[lo][-1], nxt[hi][0])
            else:
                sl.step(k, c, d, cur[s], prev[s], nxt[s], sl.blocks[0])
            if multi:
                ev = torch.cuda.Event()
                ev.record(sl.torch_stream)
                events[s] = ev
        done = events
        prev, cur = cur, nxt
    total = None
    for s in sorted(by_id):
        if multi:
            torch.cuda.current_stream(slabs[0].device).wait_stream(by_id[s].torch_stream)
        z = by_id[s].reduce().to(slabs[0].device)
        total = z if total is None else total + z
    return total


def run_rowpartition(slabs, plan, c, d, degree, mode, group=None, rank_of_slab=None, overlap=None):
    """Drive the recurrence over local slab objects (DeviceSlab or a CPU
    stand-in with the same interface: .blocks (3 ghosted blocks, block 0 holds
    the probes), .step(k, c, d, cur, prev, next, v0), .reduce(); optionally
    .parts / .step_part(name, ...) for the boundary / interior split).

    With ``overlap`` (default: when slabs live on several ranks) and slabs
    that can split (>= 3 planes each), every step runs the boundary planes,
    starts the halo exchange on a communication stream (CUDA slabs) and runs
    the interior planes while it is in flight.

    Returns the per-probe moments of the whole grid (sum over all slabs,
    all-reduced over ``group`` when slabs live on several ranks)."""
    import torch
    import torch.distributed as dist

    steps = (degree + 1) // 2 if mode == _native.SDB_CHEB_DOUBLING else degree
    if overlap is None:
        overlap = rank_of_slab is not None
    ids = [sl.s for sl in slabs]
    full = hasattr(slabs[0], "plane_doubles")  # full-size z-march blocks (PlaneSlab)

    def exchange_halo(nxt):
        if full:
            plane_exchange(slabs, plan, nxt, group, rank_of_slab)
        else:
            halo_exchange(ids, plan, nxt, group, rank_of_slab)

    split = overlap and steps > 1 and all(getattr(sl, "parts", None) for sl in slabs)
    devs = {getattr(sl, "device", None) for sl in slabs}
    dev = next(iter(devs))
    if split and len(devs) > 1:
        split = False  # one compute stream per process: the split needs the slabs on one device
    cuda = split and isinstance(dev, int)
    if cuda:
        compute = slabs[0].torch_stream
        comm = torch.cuda.Stream(device=dev)
    for sl in slabs:  # which partial buffers this run fills (reduce() sums exactly those)
        if hasattr(sl, "used"):
            sl.used.clear()
        if hasattr(sl, "split_used"):
            sl.split_used = False
    cur = {sl.s: sl.blocks[0] for sl in slabs}
    prev = {sl.s: None for sl in slabs}
    for k in range(max(steps, 1)):
        nxt = {sl.s: sl.blocks[1] if k == 0 else (sl.blocks[2] if k == 1 else prev[sl.s]) for sl in slabs}
        exchange = steps > 0 and k + 1 < steps
        if not split:
            for sl in slabs:
                sl.step(k, c, d, cur[sl.s], prev[sl.s], nxt[sl.s], sl.blocks[0])
            if exchange:
                exchange_halo(nxt)
        else:
            if cuda and k > 0:
                compute.wait_stream(comm)  # ghosts of w_k have landed
            for sl in slabs:
                for part in ("lo", "hi"):
                    sl.step_part(part, k, c, d, cur[sl.s], prev[sl.s], nxt[sl.s], sl.blocks[0])
            if exchange:
                if cuda:
                    comm.wait_stream(compute)  # boundary planes of w_{k+1} are written
                    with torch.cuda.stream(comm):
                        exchange_halo(nxt)
                else:
                    exchange_halo(nxt)
            for sl in slabs:  # interior planes overlap the exchange
                sl.step_part("int", k, c, d, cur[sl.s], prev[sl.s], nxt[sl.s], sl.blocks[0])
        prev, cur = cur, nxt
    if cuda:
        compute.wait_stream(comm)
    total = None
    for sl in slabs:
        z = sl.reduce()
        total = z if total is None else total + z
    if rank_of_slab is not None:
        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)
    return total


def make_slab(op, plan, s, n_vec, degree, mode, device, source, planes=True):
    """Slab s with its probes staged: a PlaneSlab (z-march on full-size padded
    blocks) when ``planes`` and the layout applies, else a DeviceSlab."""
    import torch

    with torch.cuda.device(device):
        if planes:
            stream = ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
            info = plane_layout(device_matrix(op, device, stream), n_vec, mode)
            if info[0] > 0:
                sl = PlaneSlab(op, plan, s, n_vec, degree, mode, device, info)
                sl.stage_probes(source)
                return sl
        sl = DeviceSlab(op, plan, s, n_vec, degree, mode, device)
        ghosted_probe_block(source, 0, n_vec, op.shape, sl.z0, sl.nzl, sl.ldv, sl.blocks[0])
        return sl


def rowpartition_moments(op, interval, degree, source, n_vec, mode=_native.SDB_CHEB_DOUBLING, n_slabs=None,
                         group=None, device=None, devices=None, exchange="p2p", overlap=None, layout="auto"):
    """Per-probe moments of (A - cI)/d for a periodic StencilOperator with the
    z-planes row-partitioned: one slab per rank of ``group`` (NCCL send/recv of
    the halo planes), or ``n_slabs`` slabs in this process spread over
    ``devices`` (default: the one device) with the halo pushed by the step
    kernels themselves over peer memory (``exchange="p2p"``; ``"copy"``: the
    step kernels plus device-to-device plane copies).  ``overlap``: split each
    step so the exchange runs beside the interior planes (default: only across
    ranks -- on one device the plane copies are cheaper than the split, which
    measured +8 % per step at 256^3).  ``layout``: "planes" (full-size z-march
    blocks, PlaneSlab), "slabs" (ghosted slab blocks, DeviceSlab) or "auto"
    (planes for the copy / NCCL exchange when the z-march applies).  Returns a
    (n_vec, degree+1) tensor on the first device."""
    import torch
    import torch.distributed as dist

    if not isinstance(op, StencilOperator) or getattr(op, "z_ghost", False):
        raise TypeError("row partition needs a periodic StencilOperator")
    if not 1 <= n_vec <= _native.SDB_MAX_BATCH:
        raise ValueError("row-partitioned moments take one probe batch (n_vec <= 256)")
    device = E.require_cuda(device)
    c, d = float(interval.center), float(interval.halfwidth)
    nz = op.shape[2]
    if group is not None or (dist.is_available() and dist.is_initialized() and n_slabs is None):
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        plan = SlabPlan(nz, world)
        local = [rank]
        rank_of_slab = lambda s: s  # noqa: E731
    else:
        plan = SlabPlan(nz, n_slabs or 1)
        local = list(range(plan.n_slabs))
        rank_of_slab = None
    if min(plan.planes(s)[1] for s in range(plan.n_slabs)) < 1:
        raise ValueError("more slabs than z-planes")
    devs = [device] if (devices is None or rank_of_slab is not None) else [int(x) for x in devices]
    use_planes = layout in ("planes", "auto")
    slabs = [make_slab(op, plan, s, n_vec, degree, mode, devs[s % len(devs)], source, use_planes) for s in local]
    with torch.cuda.device(device):
        if rank_of_slab is None and exchange == "p2p":
            return run_rowpartition_p2p(slabs, plan, c, d, degree, mode)
        if overlap is None:
            overlap = rank_of_slab is not None
        return run_rowpartition(slabs, plan, c, d, degree, mode, group if rank_of_slab else None, rank_of_slab,
                                overlap=overlap)


def prepare_rowpartition(op, interval, degree, source, n_vec, mode=_native.SDB_CHEB_DOUBLING, group=None,
                         device=None, probes_host=None):
    """Allocate this rank's slab (ghosted blocks, probes staged).  Returns
    (slabs, plan, rank_of_slab); run with ``run_rowpartition``."""
    import torch
    import torch.distributed as dist

    device = E.require_cuda(device)
    nz = op.shape[2]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    plan = SlabPlan(nz, world)
    sl = make_slab(op, plan, rank, n_vec, degree, mode, device, source, True)
    return [sl], plan, ((lambda s: s) if world > 1 else None)


def estimate_dos_rowpartition(op, interval, method, degree, source, n_vec, grid_points=200, product_formula=True,
                              group=None, device=None):
    """KPM DOS of a periodic stencil with the z-planes row-partitioned over the
    ranks of ``group`` (collective; every rank returns the same estimate)."""
    import torch

    from .compare import GPU_METHODS
    from .density import SpectralDensityEstimate, unit_grid
    from .errors import NumericalFailure

    if method not in ("kpm", "kpm-jackson"):
        raise ValueError(f"row partition supports kpm / kpm-jackson (GPU methods: {GPU_METHODS})")
    device = E.require_cuda(device)
    mode = _native.SDB_CHEB_DOUBLING if product_formula else _native.SDB_CHEB_DIRECT
    slabs, plan, ros = prepare_rowpartition(op, interval, degree, source, n_vec, mode, group, device)
    zeta_pp = run_rowpartition(slabs, plan, float(interval.center), float(interval.halfwidth), degree, mode,
                               group if ros else None, ros)
    grid = unit_grid(grid_points)
    zeta_dev, flag = E.mean_moments(zeta_pp, device)
    damp = _native.SDB_DAMP_JACKSON if method == "kpm-jackson" else _native.SDB_DAMP_NONE
    _, values, density = E.kpm_density_device(zeta_dev, degree, op.dim, damp, E.to_device(grid, device),
                                              float(interval.halfwidth), device)
    packed = torch.cat([zeta_dev, values, density, flag.to(torch.float64)]).cpu().numpy()
    m1, g = degree + 1, len(grid)
    if packed[-1] != 0.0 or not np.all(np.isfinite(packed[:m1])):
        raise NumericalFailure(E.SPECTRUM_ESCAPE_HINT)
    est = SpectralDensityEstimate.from_parts(grid, packed[m1:m1 + g], interval.from_unit(grid),
                                             packed[m1 + g:m1 + 2 * g], interval, method=method,
                                             params={"degree": degree, "moments": packed[:m1], "M": degree,
                                                     "n_vec": n_vec, "slabs": plan.n_slabs})
    if method == "kpm-jackson":
        est.params["damping"] = "jackson"
    return est

"""CPU stand-in for rowpart.DeviceSlab (test infrastructure only): the same
interface, with the step restated in NumPy on the ghosted slab blocks."""

import numpy as np
import torch

from paper_1308_5467_b200.distributed import shard_range


class NumpySlab:
    def __init__(self, op, plan, s, n_vec, degree, doubling=True):
        self.s = s
        self.z0, self.nzl = plan.planes(s)
        nx, ny, nz = op.shape
        self.nx, self.ny, self.nxy = nx, ny, nx * ny
        self.offsets, self.weights = op.offsets, op.weights
        self.diag = op.diag.reshape(nz, ny, nx)[self.z0:self.z0 + self.nzl]
        self.n_vec, self.degree, self.doubling = n_vec, degree, doubling
        shape = (self.nzl + 2, self.nxy, n_vec)
        self.blocks = [torch.zeros(shape, dtype=torch.float64) for _ in range(3)]
        self.raw = np.zeros((degree + 1, n_vec))
        # boundary / interior split, as rowpart.DeviceSlab.parts
        self.parts = {"lo": (0, 1), "int": (1, self.nzl - 1), "hi": (self.nzl - 1, self.nzl)} if self.nzl >= 3 else {}

    def step_part(self, name, k, c, d, cur, prev, nxt, v0):
        self.step(k, c, d, cur, prev, nxt, v0, planes=self.parts[name])

    def _own(self, t):
        return t[1:-1].numpy().reshape(self.nzl, self.ny, self.nx, self.n_vec)

    def step(self, k, c, d, cur, prev, nxt, v0, planes=None):
        g = cur.numpy().reshape(self.nzl + 2, self.ny, self.nx, self.n_vec)
        x = g[1:-1]
        y = self.diag[..., None] * x
        for (dx, dy, dz), w in zip(self.offsets, self.weights):
            nb = g[1 + dz:1 + dz + self.nzl]
            nb = np.roll(np.roll(nb, -dy, axis=1), -dx, axis=2)
            y = y + w * nb
        t = (y - c * x) / d
        if k == 0:
            wn = t
        else:
            wn = 2.0 * t - self._own(prev)
        a, b = planes if planes is not None else (0, self.nzl)
        wn, x = wn[a:b], x[a:b]
        nxt[1 + a:1 + b] = torch.from_numpy(wn.reshape(b - a, self.nxy, self.n_vec))
        red = lambda a, b: np.einsum("zyxl,zyxl->l", a, b)  # noqa: E731
        if self.doubling:
            if k == 0:
                self.raw[0] += red(x, x)
            if 2 * k + 1 <= self.degree:
                self.raw[2 * k + 1] += red(wn, x)
            if 2 * k + 2 <= self.degree:
                self.raw[2 * k + 2] += red(wn, wn)
        else:
            p = self._own(v0)[a:b]
            if k == 0:
                self.raw[0] += red(p, p)
            self.raw[k + 1] += red(p, wn)

    def reduce(self):
        z = self.raw.copy()
        if self.doubling:
            for k in range(2, self.degree + 1):
                z[k] = 2.0 * self.raw[k] - self.raw[k % 2]
        return torch.from_numpy(z.T.copy())


def fill_probes(slab, probes, parent_shape):
    nx, ny, nz = parent_shape
    planes = [(slab.z0 - 1) % nz] + list(range(slab.z0, slab.z0 + slab.nzl)) + [(slab.z0 + slab.nzl) % nz]
    v = probes.reshape(probes.shape[0], nz, nx * ny)[:, planes]  # (n_vec, nzl+2, nxy)
    slab.blocks[0].copy_(torch.from_numpy(np.ascontiguousarray(v.transpose(1, 2, 0))))


class NumpyPlaneSlab:
    """CPU stand-in for rowpart.PlaneSlab: full-size blocks (nz, nx*ny*n_vec)
    of the whole grid, NaN outside the probes block until written, the step
    restated in NumPy on the planes [z_lo, z_hi) with periodic z neighbours
    read from the full block (so a missing halo plane shows up as NaN)."""

    def __init__(self, op, plan, s, n_vec, degree, doubling=True):
        self.s = s
        self.z0, self.nzl = plan.planes(s)
        nx, ny, nz = op.shape
        self.nx, self.ny, self.nz = nx, ny, nz
        self.offsets, self.weights = op.offsets, op.weights
        self.diag = op.diag.reshape(nz, ny, nx)
        self.n_vec, self.degree, self.doubling = n_vec, degree, doubling
        self.plane_doubles = nx * ny * n_vec
        self.blocks = [torch.full((nz, self.plane_doubles), float("nan"), dtype=torch.float64) for _ in range(3)]
        z0, z1 = self.z0, self.z0 + self.nzl
        self.parts = {"lo": (z0, z0 + 1), "int": (z0 + 1, z1 - 1), "hi": (z1 - 1, z1)} if self.nzl >= 3 else {}
        self.raw = {}
        self.used = set()

    def _grid(self, t):
        return t.numpy().reshape(self.nz, self.ny, self.nx, self.n_vec)

    def step(self, k, c, d, cur, prev, nxt, v0):
        self._planes("all", self.z0, self.z0 + self.nzl, k, c, d, cur, prev, nxt, v0)

    def step_part(self, name, k, c, d, cur, prev, nxt, v0):
        self._planes(name, *self.parts[name], k, c, d, cur, prev, nxt, v0)

    def _planes(self, name, z_lo, z_hi, k, c, d, cur, prev, nxt, v0):
        self.used.add(name)
        raw = self.raw.setdefault(name, np.zeros((self.degree + 1, self.n_vec)))
        g = self._grid(cur)
        zs = np.arange(z_lo, z_hi)
        x = g[zs]
        y = self.diag[zs][..., None] * x
        for (dx, dy, dz), w in zip(self.offsets, self.weights):
            nb = g[(zs + dz) % self.nz]
            nb = np.roll(np.roll(nb, -dy, axis=1), -dx, axis=2)
            y = y + w * nb
        t = (y - c * x) / d
        wn = t if k == 0 else 2.0 * t - self._grid(prev)[zs]
        self._grid(nxt)[zs] = wn
        red = lambda a, b: np.einsum("zyxl,zyxl->l", a, b)  # noqa: E731
        if self.doubling:
            if k == 0:
                raw[0] += red(x, x)
            if 2 * k + 1 <= self.degree:
                raw[2 * k + 1] += red(wn, x)
            if 2 * k + 2 <= self.degree:
                raw[2 * k + 2] += red(wn, wn)
        else:
            p = self._grid(v0)[zs]
            if k == 0:
                raw[0] += red(p, p)
            raw[k + 1] += red(p, wn)

    def reduce(self):
        total = None
        for name in sorted(self.used):
            z = self.raw[name].copy()
            if self.doubling:
                for k in range(2, self.degree + 1):
                    z[k] = 2.0 * self.raw[name][k] - self.raw[name][k % 2]
            total = z if total is None else total + z
        self.raw = {}
        return torch.from_numpy(total.T.copy())


def fill_plane_probes(slab, probes):
    """Probes (n_vec, n) -> the full-size probe block (every plane valid)."""
    slab.blocks[0].copy_(torch.from_numpy(np.ascontiguousarray(probes.T)).reshape(slab.nz, -1))

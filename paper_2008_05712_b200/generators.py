"""Synthetic inputs for the hot path (host-side numpy; not the measured path).

* ``gen_particles`` reproduces the reference generator draw for draw
  (hr/workloads/nbody.py:34-49: uniform box plus <=8 Gaussian clumps, masses
  U(0.5, 1.5)), so the same seed yields the same particles.
* ``gen_plummer`` is new (no reference generator).
* ``gen_md_system`` reproduces hr/workloads/md.py:76-108 (2-D patch grid).
* ``gen_lj_fcc`` is new: FCC lattice at reduced density, Maxwell-Boltzmann
  velocities with zero net momentum.

``fp32_exact`` rounds positions/masses to float32-representable float64 so the
float64 oracle and the FP32 device path consume identical values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ParticleSet:
    positions: np.ndarray  # (n, dim) float64, within [0, box)
    masses: np.ndarray  # (n,) float64
    velocities: np.ndarray  # (n, dim)
    box: float


def gen_particles(n: int, seed: int, clustering: float = 0.0, dim: int = 2, box: float = 1.0) -> ParticleSet:
    """Same draws as hr/workloads/nbody.py:34-49."""
    if n < 1:
        raise ValueError("need at least one particle")
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, box, size=(n, dim))
    k = int(round(n * clustering))
    if k > 0:
        nclump = max(1, min(8, k))
        centers = rng.uniform(0.0, box, size=(nclump, dim))
        which = rng.integers(0, nclump, size=k)
        jitter = rng.normal(0.0, 0.02 * box, size=(k, dim))
        pos[:k] = (centers[which] + jitter) % box
    masses = rng.uniform(0.5, 1.5, size=n)
    return ParticleSet(pos, masses, np.zeros((n, dim)), box)


def gen_plummer(n: int, seed: int = 42, a: float = 0.0225, center: float = 0.5, rmax_factor: float = 20.0,
                box: float = 1.0) -> ParticleSet:
    """Plummer sphere (scale a) truncated at r <= rmax_factor*a, centred in the
    unit box, equal masses 1/n."""
    rng = np.random.default_rng(seed)
    out = np.empty((0, 3))
    rmax = rmax_factor * a
    while out.shape[0] < n:
        m = max(1024, int(1.2 * (n - out.shape[0])))
        u = rng.uniform(0.0, 1.0, size=m)
        u = np.clip(u, 1e-300, None)
        r = a / np.sqrt(u ** (-2.0 / 3.0) - 1.0)
        g = rng.normal(size=(m, 3))
        g /= np.linalg.norm(g, axis=1, keepdims=True)
        keep = r <= rmax
        out = np.vstack([out, center + r[keep, None] * g[keep]])
    pos = out[:n]
    masses = np.full(n, 1.0 / n)
    return ParticleSet(pos, masses, np.zeros((n, 3)), box)


def fp32_exact(ps: ParticleSet) -> ParticleSet:
    """Round to float32-representable values kept inside [0, box)."""
    pos = ps.positions.astype(np.float32)
    hi = np.nextafter(np.float32(ps.box), np.float32(0.0))
    pos = np.clip(pos, np.float32(0.0), hi).astype(np.float64)
    m = ps.masses.astype(np.float32).astype(np.float64)
    return ParticleSet(pos, m, ps.velocities.copy(), ps.box)


# ---------------------------------------------------------------------------
# molecular dynamics inputs
# ---------------------------------------------------------------------------

def gen_md_system(grid_dim, particles_per_patch, cutoff, seed, patch_size=None):
    """Same draws as hr/workloads/md.py:76-108.  Returns (positions,
    velocities, patch_of, rows, cols, patch_size)."""
    rows, cols = grid_dim
    ps_ = cutoff if patch_size is None else patch_size
    if ps_ < cutoff:
        raise ValueError("patch size must cover the cutoff distance")
    rng = np.random.default_rng(seed)
    n = rows * cols * particles_per_patch
    pr = rng.integers(0, rows, size=n)
    pc = rng.integers(0, cols, size=n)
    off = rng.uniform(0.0, ps_, size=(n, 2))
    pos = np.column_stack([pr * ps_, pc * ps_]) + off
    vel = rng.normal(0.0, 0.35 * ps_, size=(n, 2))
    return pos, vel, (pr * cols + pc).astype(np.int64), rows, cols, ps_


@dataclass
class LJSystem:
    positions: np.ndarray  # (n, 3) float64 (float32-exact)
    velocities: np.ndarray  # (n, 3)
    box: float  # y / z box (and x for repeat_x = 1)
    cells: int  # cells per y / z dimension
    cell_size: float
    rc: float = 2.5
    eps: float = 1.0
    sigma: float = 1.0
    dt: float = 0.005
    repeat_x: int = 1  # the lattice is repeated along x (slab decompositions)

    @property
    def cells_xyz(self):
        return (self.cells * self.repeat_x, self.cells, self.cells)

    @property
    def box_xyz(self):
        # the device's box: cells x cell size per dimension
        return tuple(c * self.cell_size for c in self.cells_xyz)


def gen_lj_fcc(lattice_cells: int = 30, rho: float = 0.8442, temperature: float = 1.44, seed: int = 7,
               rc: float = 2.5, dt: float = 0.005, repeat_x: int = 1) -> LJSystem:
    """FCC lattice, 4 atoms per unit cell, lattice_cells^3 unit cells (x
    lattice_cells * repeat_x along x)."""
    a = (4.0 / rho) ** (1.0 / 3.0)
    box = lattice_cells * a
    basis = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]])
    g = np.arange(lattice_cells)
    gx = np.arange(lattice_cells * repeat_x)
    cell = np.stack(np.meshgrid(gx, g, g, indexing="ij"), axis=-1).reshape(-1, 3)
    pos = ((cell[:, None, :] + basis[None, :, :] + 0.25) * a).reshape(-1, 3)
    ncell = max(3, int(np.floor(box / rc)))
    cs = box / ncell
    bx = (ncell * repeat_x) * cs if repeat_x > 1 else box
    pos = pos.astype(np.float32).astype(np.float64) % np.array([bx, box, box])
    rng = np.random.default_rng(seed)
    vel = rng.normal(0.0, np.sqrt(temperature), size=pos.shape)
    vel -= vel.mean(axis=0)
    vel = vel.astype(np.float32).astype(np.float64)
    return LJSystem(pos, vel, box, ncell, cs, rc=rc, dt=dt, repeat_x=repeat_x)

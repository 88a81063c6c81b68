"""Cell-pair molecular dynamics on B200 (mirrors hr/workloads/md.py).

The 2-D soft-repulsion patch MD keeps the reference's API: ``PatchGrid``
(24-46), ``neighbor_pairs`` (49-73), ``gen_md_system`` (76-108),
``pair_work`` (111-118), ``compute_forces`` (121-163) and ``md_step``
(166-190); the force evaluation and the integrator run in libgcharm's
cell-pair kernels (csrc/md.cu) with the reference's float64 arithmetic.
``LJSystem`` is the 3-D cutoff Lennard-Jones workload of BASELINE.json
configs[1]/[4] (no reference counterpart): it stays resident in HBM and
``run(steps)`` replays a CUDA graph of whole md_step iterations.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .generators import LJSystem as _LJInput
from .generators import gen_lj_fcc  # noqa: F401

_NEIGHBOR_STEPS = ((0, 1), (1, -1), (1, 0), (1, 1))
LAW_SOFT, LAW_LJ = 0, 1


@dataclass
class PatchGrid:
    rows: int
    cols: int
    patch_size: float
    cutoff: float
    positions: np.ndarray  # (n, 2)
    velocities: np.ndarray  # (n, 2)
    patch_of: np.ndarray  # (n,) linear patch index

    @property
    def n_patches(self) -> int:
        return self.rows * self.cols

    @property
    def box(self):
        return self.rows * self.patch_size, self.cols * self.patch_size

    def populations(self) -> np.ndarray:
        return np.bincount(self.patch_of, minlength=self.n_patches)

    def particles_in(self, patch: int) -> np.ndarray:
        return np.nonzero(self.patch_of == patch)[0]


def neighbor_pairs(rows: int, cols: int, periodic: bool = False):
    """Self pairs plus each touching patch pair once (md.py:49-73)."""
    out, seen = [], set()
    for r in range(rows):
        for c in range(cols):
            p = r * cols + c
            out.append((p, p))
            seen.add((p, p))
            for dr, dc in _NEIGHBOR_STEPS:
                rr, cc = r + dr, c + dc
                if periodic:
                    rr, cc = rr % rows, cc % cols
                elif not (0 <= rr < rows and 0 <= cc < cols):
                    continue
                q = rr * cols + cc
                key = (min(p, q), max(p, q))
                if key not in seen:
                    seen.add(key)
                    out.append((p, q))
    return out


def gen_md_system(grid_dim, particles_per_patch, cutoff, seed, patch_size=None):
    from .generators import gen_md_system as _gen
    pos, vel, patch_of, rows, cols, ps_ = _gen(grid_dim, particles_per_patch, cutoff, seed, patch_size)
    grid = PatchGrid(rows, cols, ps_, cutoff, pos, vel, patch_of)
    return grid, pair_work(grid)


def pair_work(grid: PatchGrid, periodic: bool = False):
    pops = grid.populations()
    out = []
    for a, b in neighbor_pairs(grid.rows, grid.cols, periodic):
        items = int(pops[a]) * int(pops[b])
        if items > 0:
            out.append((a, b, items))
    return out


class _Device:
    """A libgcharm gc_md handle."""

    def __init__(self):
        self._ctx = L.context()
        self.handle = C.c_void_p()
        L.call("gc_md_create", self._ctx.handle, C.byref(self.handle))

    def __del__(self):
        try:
            if self.handle:
                L.load().gc_md_destroy(self.handle)
        except Exception:
            pass

    def set(self, pos, vel, cell_of, dims, cell_size, periodic, law, params):
        pos = L.f64(pos)
        n, d = pos.shape
        v = L.f64(vel) if vel is not None else None
        co = L.i64(cell_of) if cell_of is not None else None
        dm = L.i64(dims)
        pr = L.f64(params)
        L.call("gc_md_set_system", self.handle, n, d, L.ptr(pos, L.f64p), L.ptr(v, L.f64p) if v is not None else None,
               L.ptr(co, L.i64p) if co is not None else None, L.ptr(dm, L.i64p), float(cell_size), int(bool(periodic)),
               int(law), L.ptr(pr, L.f64p))
        self.n, self.dim = n, d

    def forces(self, energy=False):
        f = np.zeros((self.n, self.dim))
        e = np.zeros(self.n) if energy else None
        L.call("gc_md_forces", self.handle, L.ptr(f, L.f64p), L.ptr(e, L.f64p) if e is not None else None)
        return (f, e) if energy else f

    def run(self, steps, dt):
        L.call("gc_md_run", self.handle, int(steps), float(dt))

    def state(self):
        p, v = np.zeros((self.n, self.dim)), np.zeros((self.n, self.dim))
        c = np.zeros(self.n, np.int64)
        L.call("gc_md_get_state", self.handle, L.ptr(p, L.f64p), L.ptr(v, L.f64p), L.ptr(c, L.i64p))
        return p, v, c

    def elapsed_ms(self) -> float:
        out = np.zeros(1)
        L.call("gc_md_elapsed", self.handle, L.ptr(out, L.f64p))
        return float(out[0])


def _grid_device(grid: PatchGrid, stiffness: float, periodic: bool) -> _Device:
    dev = _Device()
    dev.set(grid.positions, grid.velocities, grid.patch_of, (grid.rows, grid.cols, 1), grid.patch_size, periodic,
            LAW_SOFT, (grid.cutoff, stiffness, 0.0))
    return dev


def compute_forces(grid: PatchGrid, stiffness: float = 25.0, periodic: bool = False) -> np.ndarray:
    """md.py:121-163 on the GPU (float64, reference cutoff decisions)."""
    return _grid_device(grid, stiffness, periodic).forces()


def md_step(grid: PatchGrid, dt: float, stiffness: float = 25.0, periodic: bool = False) -> PatchGrid:
    """md.py:166-190 on the GPU: forces, v += F dt, x += v dt, walls or wrap,
    patch reassignment (numpy floor_divide semantics)."""
    dev = _grid_device(grid, stiffness, periodic)
    dev.run(1, dt)
    grid.positions, grid.velocities, grid.patch_of = dev.state()
    return grid


class LJSystem:
    """Device-resident 3-D cutoff Lennard-Jones system on a periodic cell grid
    (cells of side >= rc; the md_step structure in 3-D)."""

    def __init__(self, inp: _LJInput):
        self.inp = inp
        self.dev = _Device()
        self.dims = inp.cells_xyz
        self.dev.set(inp.positions, inp.velocities, None, self.dims, inp.cell_size, True, LAW_LJ,
                     (inp.rc, inp.eps, inp.sigma))
        self.n = inp.positions.shape[0]

    def forces(self):
        """(forces (n, 3), per-atom energy (n,)) on the current positions."""
        return self.dev.forces(energy=True)

    def run(self, steps: int, dt: float | None = None):
        self.dev.run(steps, self.inp.dt if dt is None else dt)
        return self.dev.elapsed_ms()

    def state(self):
        return self.dev.state()

    def task_count(self) -> int:
        """Cell-pair work requests per step: self + 13 half-shell pairs per cell."""
        return 14 * self.dims[0] * self.dims[1] * self.dims[2]


# -- closed-loop MD on the device ---------------------------------

@dataclass
class MDParams:
    """hr/workloads/md.py:193-206 (the timing fields drive only the
    reference's simulated clock; the device loop runs as fast as it can)."""
    rows: int = 10
    cols: int = 10
    particles_per_patch: int = 24
    cutoff: float = 1.0
    steps: int = 12
    dt: float = 0.08
    stiffness: float = 25.0
    seed: int = 7
    ready_cost: float = 0.01
    migrate_cost: float = 2.0
    bytes_per_item: int = 16
    periodic: bool = False


@dataclass
class ClosedLoopResult:
    """Per-step counts of the device's message-driven loop and the runtime's
    invocation totals (hr/runtime.py InvocationRecord, per entry method)."""
    work_requests: np.ndarray  # per step: len(pair_work) submitted
    interact_messages: np.ndarray  # per step: "interact" messages delivered
    completions: np.ndarray  # per step: work_done messages into the barrier
    barriers: int  # step_barrier invocations
    device_ms: float

    @property
    def invocations(self) -> dict:
        return {"interact": int(self.work_requests.sum()), "work_done": int(self.completions.sum()),
                "step_barrier": int(self.barriers)}


class MDWorkload:
    """Closed-loop MD run (md.py:209-271) executed on the device: step k+1's
    requests only arrive after step k's barrier, all inside one persistent
    kernel (csrc/md_loop.cu).  ``run()`` replaces ``setup(tl)`` + ``tl.run()``
    of the simulator; ``grid`` and ``step`` end as the reference's do."""

    kernel_class = "md"

    def __init__(self, params: MDParams):
        self.params = params
        self.grid, _ = gen_md_system((params.rows, params.cols), params.particles_per_patch, params.cutoff,
                                     params.seed)
        self.step = 0
        self._ctx = L.context()
        self.handle = C.c_void_p()
        L.call("gc_mdloop_create", self._ctx.handle, C.byref(self.handle))

    def __del__(self):
        try:
            if self.handle:
                L.load().gc_mdloop_destroy(self.handle)
        except Exception:
            pass

    def kernel_classes(self) -> list:
        return ["md"]

    def topology(self) -> tuple:
        """(patches, pair chares, compute_forces segments)."""
        out = np.zeros(3, np.int64)
        L.call("gc_mdloop_topology", self.handle, L.ptr(out, L.i64p))
        return tuple(int(x) for x in out)

    def phases_ns(self) -> np.ndarray:
        """(steps, 5) ns per phase of the last run: counts + scans, scatter,
        patch sort / gather / messages, execution + barrier, md_step."""
        out = np.zeros((max(self.params.steps, 1), 5))
        L.call("gc_mdloop_phases", self.handle, L.ptr(out, L.f64p))
        return out[:self.params.steps]

    def run(self) -> ClosedLoopResult:
        p, g = self.params, self.grid
        pos, vel, pc = L.f64(g.positions), L.f64(g.velocities), L.i64(g.patch_of)
        L.call("gc_mdloop_set", self.handle, len(pos), L.ptr(pos, L.f64p), L.ptr(vel, L.f64p), L.ptr(pc, L.i64p),
               int(g.rows), int(g.cols), float(g.patch_size), float(g.cutoff), float(p.stiffness),
               int(bool(p.periodic)))
        stats = np.zeros((max(p.steps, 1), 4), np.int64)
        L.call("gc_mdloop_run", self.handle, int(p.steps), float(p.dt), L.ptr(stats, L.i64p))
        n = len(pos)
        g.positions, g.velocities, g.patch_of = np.zeros((n, 2)), np.zeros((n, 2)), np.zeros(n, np.int64)
        L.call("gc_mdloop_get_state", self.handle, L.ptr(g.positions, L.f64p), L.ptr(g.velocities, L.f64p),
               L.ptr(g.patch_of, L.i64p))
        ms = np.zeros(1)
        L.call("gc_mdloop_elapsed", self.handle, L.ptr(ms, L.f64p))
        stats = stats[:p.steps]
        self.step = int(stats[:, 3].sum())
        return ClosedLoopResult(stats[:, 0].copy(), stats[:, 1].copy(), stats[:, 2].copy(), self.step, float(ms[0]))

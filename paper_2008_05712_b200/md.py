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


# -- configs[4]: force work arriving at a varying generation rate ----------------

class LJColumnPhase:
    """One LJ force phase as work requests arriving at a varying rate,
    combined by the batcher's trigger and launched column batch by column
    batch (BASELINE configs[4]: "varying task-generation rate").

    Work request = one column of KZ home cells (the column kernel's unit; its
    forces read the 3 x 3 x (KZ + 2) neighbour cells).  Its arrival is the
    last "interact" input of its cells: start + ready_cost x the largest
    population among those cells (hr/workloads/md.py:236-254), plus lognormal
    lulls between pieces of the column order (NBodyWorkload._schedule,
    hr/workloads/nbody.py:285-301).  The trigger (hr/aggregator.py:41-110,
    evaluated on the device, gc_batcher_trigger_device) cuts the FIFO of
    columns into combined launches of at most max_size requests (the column
    kernel's occupancy x SMs); each batch is one gc_md_forces_columns launch.
    Forces are those of the whole-system launch bit for bit (the same
    per-column arithmetic)."""

    def __init__(self, system: "LJSystem", max_size: int | None = None, ready_cost: float = 0.01,
                 pieces: int = 16, piece_gap: float = 4.0, seed: int = 7, timeout_factor: float = 2.0,
                 tick: float = 1.0):
        from .aggregator import compute_max_size
        from .devicesim import b200_device_spec, b200_kernel_spec
        self.sys = system
        info = np.zeros(3, np.int64)
        L.call("gc_md_columns", system.dev.handle, L.ptr(info, L.i64p))
        if info[0] == 0:
            raise ValueError("the column kernel does not apply to this system (needs >= 3 cells per dimension)")
        self.ncol, self.kz, self.ncz = int(info[0]), int(info[1]), int(info[2])
        if max_size is None:
            max_size = compute_max_size(b200_kernel_spec("md_column"), b200_device_spec())
        self.max_size, self.timeout_factor, self.tick = int(max_size), float(timeout_factor), float(tick)
        self.ready_cost, self.pieces, self.piece_gap, self.seed = ready_cost, pieces, piece_gap, seed

    def arrivals(self, positions) -> tuple:
        """(column order by arrival, arrival times) for the current positions."""
        nx, ny, nz = self.sys.dims
        cell = self.sys.inp.cell_size
        c = np.clip(np.floor(positions / cell).astype(np.int64), 0, np.array([nx - 1, ny - 1, nz - 1]))
        pop = np.bincount((c[:, 0] * ny + c[:, 1]) * nz + c[:, 2], minlength=nx * ny * nz).reshape(nx, ny, nz)
        # largest population over each cell's 3 x 3 x 3 neighbourhood (periodic)
        m = pop.copy()
        for ax in range(3):
            m = np.maximum(np.maximum(m, np.roll(m, 1, axis=ax)), np.roll(m, -1, axis=ax))
        kz, ncz = self.kz, self.ncz
        colmax = np.zeros((nx, ny, ncz), np.int64)
        for zb in range(ncz):
            colmax[:, :, zb] = m[:, :, zb * kz:(zb + 1) * kz].max(axis=2)
        ready = self.ready_cost * colmax.reshape(-1).astype(float)
        # lulls between pieces of the column order (lognormal, as _schedule)
        rng = np.random.default_rng(self.seed + 1)
        per_piece = max(1, -(-self.ncol // self.pieces))
        lull = np.zeros(self.ncol)
        for k in range(1, self.pieces):
            lull[k * per_piece:] += self.piece_gap * float(rng.lognormal(0.0, 1.0))
        t = ready + lull
        order = np.argsort(t, kind="stable")
        return order.astype(np.int32), t[order]

    def events(self, t):
        """Trigger events: every arrival, and a poll at each multiple of `tick`
        (the timeline's ticks while requests are pending, hr/timeline.py:391-399;
        a poll with nothing pending is a no-op); arrivals at a tick come first."""
        ticks = np.arange(np.floor(t[0] / self.tick) + 1, np.floor(t[-1] / self.tick) + 2) * self.tick if len(t) else []
        times = np.concatenate([t, ticks])
        poll = np.concatenate([np.zeros(len(t), np.int8), np.ones(len(ticks), np.int8)])
        o = np.lexsort((poll, times))
        return times[o], poll[o]

    def run(self):
        """The phase: (forces (n, 3), energy (n,), batches [(first, count, time)], device ms)."""
        import torch

        from .executor import DeviceBatcher
        p, _, _ = self.sys.state()  # positions as last sorted on the device
        order, t = self.arrivals(p)
        ev_t, ev_p = self.events(t)
        f, c, tt = DeviceBatcher.trigger_device(self.max_size, self.timeout_factor, 0, ev_t, is_poll=ev_p)
        rest = len(order) - int(c.sum())  # end of the phase: drain in max_size chunks
        if rest:
            base = int(c.sum())
            extra = [(base + k, min(self.max_size, rest - k)) for k in range(0, rest, self.max_size)]
            f = np.concatenate([f, [e[0] for e in extra]]).astype(np.int64)
            c = np.concatenate([c, [e[1] for e in extra]]).astype(np.int64)
            tt = np.concatenate([tt, [float(t[-1])] * len(extra)])
        dev = torch.device("cuda", torch.cuda.current_device())
        cols = torch.from_numpy(order).to(dev)
        ctx = self.sys.dev._ctx
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        stream = torch.cuda.ExternalStream(ctx.stream)
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for a, k in zip(f, c):  # one combined launch per emitted batch
                L.call("gc_md_forces_columns", self.sys.dev.handle, C.c_void_p(cols.data_ptr() + 4 * int(a)), int(k))
            ev[1].record(stream)
        ev[1].synchronize()
        n = self.sys.n
        fo, e = np.zeros((n, 3)), np.zeros(n)
        L.call("gc_md_get_forces", self.sys.dev.handle, L.ptr(fo, L.f64p), L.ptr(e, L.f64p))
        return fo, e, list(zip(f.tolist(), c.tolist(), tt.tolist())), ev[0].elapsed_time(ev[1])


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

"""x-slab spatial decomposition of the cell-pair LJ MD over the GPUs of one box
(BASELINE.json configs[4]: LJ MD spatially decomposed across
B200s with a halo exchange).

The reference runs every patch pair of ``compute_forces`` / ``md_step``
(hr/workloads/md.py:121-190) in one process.  Here rank r owns the global x
cells [bounds[r], bounds[r+1]) of the periodic cell grid and keeps its atoms
resident in HBM (a gc_md slab handle, csrc/md.cu).  One step:

  1. halo: the owned atoms of the first / last owned cell plane go to the
     left / right neighbour, whose ghost planes they become;
  2. the fused cell-pair force + integrator kernel runs on the owned cells
     (ghost cells are read, never integrated), image shifts follow the GLOBAL
     periodic grid, cells are ordered by global atom id, so every force,
     cutoff decision and position is bit-identical to the whole-domain run;
  3. migration: owned atoms whose new cell left the slab move to the
     neighbour (position, velocity, global id).

The exchanges are neighbour send/recv of variable-size records (counts first),
over NCCL between GPUs (``DistTransport``), over gloo on CPU tensors in the
tests, or in-process between slabs sharing one device (``LocalTransport``).
There is no collective on the force path; per-step device time is reduced by
MAX over ranks only for reporting.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .md import LAW_LJ, _Device

GHOST, MIGRANT = 4, 8  # float64 words per packed record (1 or 2 double4)


def slab_bounds(gnx: int, k: int) -> list:
    """K + 1 cell boundaries splitting gnx x cells as evenly as possible."""
    if k < 1 or gnx < k:
        raise ValueError("need 1 <= k <= gnx")
    return [r * gnx // k for r in range(k + 1)]


def neighbours(rank: int, k: int):
    """(left, right) ranks on the periodic ring of slabs."""
    return (rank - 1) % k, (rank + 1) % k


def global_cell_x(x: np.ndarray, cell: float, gnx: int) -> np.ndarray:
    """Global x cell of positions: floor(x / cell) clamped to the grid (the
    device's md_cell_index for 3-D cells)."""
    return np.clip(np.floor(x / cell).astype(np.int64), 0, gnx - 1)


class DistTransport:
    """Neighbour exchange over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.k = dist.get_world_size(group)

    def _peer(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def exchange(self, to_left, to_right):
        """Send `to_left` to the left neighbour and `to_right` to the right one;
        return (from_left, from_right).  Tensors are (n, w) float64 on the
        transport's device; n may differ per message and may be 0."""
        import torch
        if self.k == 1:  # a single slab is its own left and right neighbour
            return to_right, to_left
        if self.dist.get_backend(self.group) == "gloo" and to_left.device.type == "cuda":
            dev = to_left.device  # gloo moves host tensors
            fl, fr = self.exchange(to_left.cpu(), to_right.cpu())
            return fl.to(dev), fr.to(dev)
        dist = self.dist
        left, right = neighbours(self.rank, self.k)
        dev, w = to_left.device, to_left.shape[1]
        # NCCL ignores tags and matches a pair's messages in issue order, and with
        # two slabs the left and right neighbour are the same rank: every rank
        # issues [send left, send right, recv right, recv left], so a peer's
        # k-th receive from us is our k-th send to it (tags kept for gloo).
        # Counts first (tag 0: travelling left, tag 1: travelling right).
        sl = torch.tensor([to_left.shape[0]], dtype=torch.int64, device=dev)
        sr = torch.tensor([to_right.shape[0]], dtype=torch.int64, device=dev)
        rl, rr = torch.zeros_like(sl), torch.zeros_like(sr)
        ops = [dist.P2POp(dist.isend, sl, self._peer(left), self.group, 0),
               dist.P2POp(dist.isend, sr, self._peer(right), self.group, 1),
               dist.P2POp(dist.irecv, rr, self._peer(right), self.group, 0),
               dist.P2POp(dist.irecv, rl, self._peer(left), self.group, 1)]
        for q in dist.batch_isend_irecv(ops):
            q.wait()
        fl = torch.empty((int(rl.item()), w), dtype=torch.float64, device=dev)
        fr = torch.empty((int(rr.item()), w), dtype=torch.float64, device=dev)
        ops = []
        if to_left.shape[0]:
            ops.append(dist.P2POp(dist.isend, to_left.contiguous(), self._peer(left), self.group, 2))
        if to_right.shape[0]:
            ops.append(dist.P2POp(dist.isend, to_right.contiguous(), self._peer(right), self.group, 3))
        if fr.shape[0]:
            ops.append(dist.P2POp(dist.irecv, fr, self._peer(right), self.group, 2))
        if fl.shape[0]:
            ops.append(dist.P2POp(dist.irecv, fl, self._peer(left), self.group, 3))
        if ops:
            for q in dist.batch_isend_irecv(ops):
                q.wait()
        if dev.type == "cuda":
            torch.cuda.synchronize(dev)  # the slab's own stream reads the received records next
        return fl, fr


    def exchange_fixed(self, send_l, cnt_l, send_r, cnt_r, recv_l, rcnt_l, recv_r, rcnt_r, stream=None):
        """Device-count exchange: fixed-capacity record buffers and their int32
        counts, all stream-ordered on `stream` (NCCL peer sends; the current
        stream waits for the receives) -- no host round trip.  recv_l gets the
        left neighbour's `send_r`, recv_r the right neighbour's `send_l`."""
        import torch
        dist = self.dist
        if self.k == 1:  # a single slab is its own left and right neighbour
            with torch.cuda.stream(stream) if stream is not None else _nullctx():
                recv_l.copy_(send_r)
                rcnt_l.copy_(cnt_r)
                recv_r.copy_(send_l)
                rcnt_r.copy_(cnt_l)
            return
        left, right = neighbours(self.rank, self.k)
        if send_l.is_cuda and dist.get_backend(self.group) == "gloo":
            self._exchange_fixed_gloo(left, right, (cnt_l, send_l, cnt_r, send_r), (rcnt_r, recv_r, rcnt_l, recv_l),
                                      stream)
            return
        # same issue order on every rank (see exchange): sends left, right, receives right, left
        ops = [dist.P2POp(dist.isend, cnt_l, self._peer(left), self.group, 0),
               dist.P2POp(dist.isend, send_l, self._peer(left), self.group, 2),
               dist.P2POp(dist.isend, cnt_r, self._peer(right), self.group, 1),
               dist.P2POp(dist.isend, send_r, self._peer(right), self.group, 3),
               dist.P2POp(dist.irecv, rcnt_r, self._peer(right), self.group, 0),
               dist.P2POp(dist.irecv, recv_r, self._peer(right), self.group, 2),
               dist.P2POp(dist.irecv, rcnt_l, self._peer(left), self.group, 1),
               dist.P2POp(dist.irecv, recv_l, self._peer(left), self.group, 3)]
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            for q in dist.batch_isend_irecv(ops):
                q.wait()  # NCCL: the current (library) stream waits; gloo: completes on the host


    def _exchange_fixed_gloo(self, left, right, sends, recvs, stream):
        """exchange_fixed for the GCHARM_DIST_BACKEND=gloo dry run: gloo moves
        host memory only, so the device buffers are staged through the host
        (synchronous; the NCCL path above has no host round trip)."""
        import torch
        dist = self.dist
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            hs = [t.cpu() for t in sends]
            hr = [torch.empty(t.shape, dtype=t.dtype) for t in recvs]
            ops = [dist.P2POp(dist.isend, hs[0], self._peer(left), self.group, 0),
                   dist.P2POp(dist.isend, hs[1], self._peer(left), self.group, 2),
                   dist.P2POp(dist.isend, hs[2], self._peer(right), self.group, 1),
                   dist.P2POp(dist.isend, hs[3], self._peer(right), self.group, 3),
                   dist.P2POp(dist.irecv, hr[0], self._peer(right), self.group, 0),
                   dist.P2POp(dist.irecv, hr[1], self._peer(right), self.group, 2),
                   dist.P2POp(dist.irecv, hr[2], self._peer(left), self.group, 1),
                   dist.P2POp(dist.irecv, hr[3], self._peer(left), self.group, 3)]
            for q in dist.batch_isend_irecv(ops):
                q.wait()
            for dst, src in zip(recvs, hr):
                dst.copy_(src)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class LocalTransport:
    """All K slabs in one process (one GPU): messages are handed over directly.
    ``exchange_all`` takes every slab's (to_left, to_right) at once."""

    def __init__(self, k: int):
        self.k = k

    def exchange_all(self, outgoing):
        out = []
        for r in range(self.k):
            left, right = neighbours(r, self.k)
            out.append((outgoing[left][1], outgoing[right][0]))
        return out

    def exchange_all_fixed(self, slabs, kind: str):
        """Device-count form for K slabs on one device (same stream): every
        slab's left receive buffer gets its left neighbour's right send."""
        for r, s in enumerate(slabs):
            left, right = neighbours(r, self.k)
            sl, sr = slabs[left].bufs[kind], slabs[right].bufs[kind]
            b = s.bufs[kind]
            b["recv_l"].copy_(sl["send_r"])
            b["cnt"][2:3].copy_(sl["cnt"][1:2])
            b["recv_r"].copy_(sr["send_l"])
            b["cnt"][3:4].copy_(sr["cnt"][0:1])


class LJSlab:
    """One rank's slab of a periodic LJ system (an ``md.LJSystem`` input)."""

    def __init__(self, inp, gx0: int, gx1: int):
        import torch
        self.torch = torch
        self.inp = inp
        self.gnx, self.ny, self.nz = (int(c) for c in inp.cells_xyz)
        self.gx0, self.gx1 = gx0, gx1
        cx = global_cell_x(inp.positions[:, 0], inp.cell_size, self.gnx)
        own = np.nonzero((cx >= gx0) & (cx < gx1))[0]
        self.dev = _Device()
        self.dev.set(inp.positions[own], inp.velocities[own], None, (gx1 - gx0 + 2, self.ny, self.nz),
                     inp.cell_size, True, LAW_LJ, (inp.rc, inp.eps, inp.sigma))
        gid = np.ascontiguousarray(own, dtype=np.int64)
        L.call("gc_md_set_slab", self.dev.handle, gx0, self.gnx, L.ptr(gid, L.i64p))
        self.device = torch.device("cuda", torch.cuda.current_device())

    def _pack(self, what: int, width: int):
        torch = self.torch
        n = np.zeros(1, np.int64)
        L.call("gc_md_pack", self.dev.handle, what, None, 0, L.ptr(n, L.i64p))
        buf = torch.empty((int(n[0]), width), dtype=torch.float64, device=self.device)
        if n[0]:
            L.call("gc_md_pack", self.dev.handle, what, C.c_void_p(buf.data_ptr()), int(n[0]), L.ptr(n, L.i64p))
        return buf

    @staticmethod
    def _ptr(t):
        return C.c_void_p(t.data_ptr()) if t.shape[0] else None

    def halo_out(self):
        """(to_left, to_right): owned atoms of the first / last owned plane."""
        return self._pack(0, GHOST), self._pack(1, GHOST)

    def set_halo(self, from_left, from_right):
        L.call("gc_md_set_ghosts", self.dev.handle, self._ptr(from_left), from_left.shape[0], self._ptr(from_right),
               from_right.shape[0])

    def advance(self, dt: float):
        L.call("gc_md_slab_step", self.dev.handle, float(dt))

    def migrants_out(self):
        return self._pack(2, MIGRANT), self._pack(3, MIGRANT)

    def take_migrants(self, from_left, from_right):
        L.call("gc_md_migrate", self.dev.handle, self._ptr(from_left), from_left.shape[0], self._ptr(from_right),
               from_right.shape[0])

    # -- device-count step (no host round trip: counts travel with the records) --
    def enable_device_counts(self, halo_cap: int | None = None):
        """Fixed-capacity message buffers for the device-count step: a plane's
        atoms (ny x nz cells) with a 2x margin, for the ghosts and the migrants."""
        torch = self.torch
        if halo_cap is None:
            per_cell = max(1.0, self.inp.positions.shape[0] / float(self.gnx * self.ny * self.nz))
            halo_cap = int(2.0 * per_cell * self.ny * self.nz) + 1024
        self.cap = int(halo_cap)
        self.stream = torch.cuda.ExternalStream(self.dev._ctx.stream) if self.device.type == "cuda" else None
        self.bufs = {}
        for kind, w in (("halo", GHOST), ("mig", MIGRANT)):
            self.bufs[kind] = {
                "send_l": torch.zeros((self.cap, w), dtype=torch.float64, device=self.device),
                "send_r": torch.zeros((self.cap, w), dtype=torch.float64, device=self.device),
                "recv_l": torch.zeros((self.cap, w), dtype=torch.float64, device=self.device),
                "recv_r": torch.zeros((self.cap, w), dtype=torch.float64, device=self.device),
                "cnt": torch.zeros(4, dtype=torch.int32, device=self.device),  # send l, send r, recv l, recv r
            }

    def _p(self, t, i=0):
        return C.c_void_p(t.data_ptr() + i * t.element_size())

    def pack_dev(self, kind: str):
        b = self.bufs[kind]
        w0 = 0 if kind == "halo" else 2
        L.call("gc_md_pack_dev", self.dev.handle, w0, self._p(b["send_l"]), self.cap, self._p(b["cnt"], 0))
        L.call("gc_md_pack_dev", self.dev.handle, w0 + 1, self._p(b["send_r"]), self.cap, self._p(b["cnt"], 1))

    def exchange_dev(self, transport: DistTransport, kind: str):
        b = self.bufs[kind]
        c = b["cnt"]
        transport.exchange_fixed(b["send_l"], c[0:1], b["send_r"], c[1:2], b["recv_l"], c[2:3], b["recv_r"], c[3:4],
                                 stream=self.stream)

    def set_halo_dev(self):
        b = self.bufs["halo"]
        L.call("gc_md_set_ghosts_dev", self.dev.handle, self._p(b["recv_l"]), self._p(b["cnt"], 2),
               self._p(b["recv_r"]), self._p(b["cnt"], 3), self.cap)

    def advance_dev(self, dt: float):
        L.call("gc_md_slab_step_dev", self.dev.handle, float(dt))

    def take_migrants_dev(self):
        b = self.bufs["mig"]
        L.call("gc_md_migrate_dev", self.dev.handle, self._p(b["recv_l"]), self._p(b["cnt"], 2),
               self._p(b["recv_r"]), self._p(b["cnt"], 3), self.cap)

    def step_dev(self, transport: DistTransport, dt: float | None = None):
        """One step with every count on the device: pack -> exchange (stream-
        ordered NCCL) -> ghosts -> forces + integrator -> migrants -> exchange ->
        migrate.  Nothing here waits for the device."""
        dt = self.inp.dt if dt is None else dt
        self.pack_dev("halo")
        self.exchange_dev(transport, "halo")
        self.set_halo_dev()
        self.advance_dev(dt)
        self.pack_dev("mig")
        self.exchange_dev(transport, "mig")
        self.take_migrants_dev()

    def step(self, transport: DistTransport, dt: float | None = None):
        dt = self.inp.dt if dt is None else dt
        self.set_halo(*transport.exchange(*self.halo_out()))
        self.advance(dt)
        self.take_migrants(*transport.exchange(*self.migrants_out()))

    def elapsed_ms(self) -> float:
        return self.dev.elapsed_ms()

    def owned(self):
        """(positions, velocities, global ids) of the owned atoms (host)."""
        n = np.zeros(1, np.int64)
        L.call("gc_md_owned", self.dev.handle, L.ptr(n, L.i64p), None, None, None)
        k = int(n[0])
        p, v, g = np.zeros((k, 3)), np.zeros((k, 3)), np.zeros(k, np.int64)
        L.call("gc_md_owned", self.dev.handle, L.ptr(n, L.i64p), L.ptr(p, L.f64p), L.ptr(v, L.f64p),
               L.ptr(g, L.i64p))
        return p, v, g


def run_local(inp, k: int, steps: int, dt: float | None = None):
    """K slabs on the current GPU, exchanged in-process; returns the assembled
    global (positions, velocities) in original atom order."""
    b = slab_bounds(inp.cells_xyz[0], k)
    slabs = [LJSlab(inp, b[r], b[r + 1]) for r in range(k)]
    tr = LocalTransport(k)
    dt = inp.dt if dt is None else dt
    for _ in range(steps):
        for s, (fl, fr) in zip(slabs, tr.exchange_all([s.halo_out() for s in slabs])):
            s.set_halo(fl, fr)
        for s in slabs:
            s.advance(dt)
        for s, (fl, fr) in zip(slabs, tr.exchange_all([s.migrants_out() for s in slabs])):
            s.take_migrants(fl, fr)
    return assemble([s.owned() for s in slabs], inp.positions.shape[0])


def run_local_dev(inp, k: int, steps: int, dt: float | None = None):
    """run_local with the device-count step (fixed-capacity messages, counts
    on the device); returns the assembled global (positions, velocities)."""
    b = slab_bounds(inp.cells_xyz[0], k)
    slabs = [LJSlab(inp, b[r], b[r + 1]) for r in range(k)]
    for s in slabs:
        s.enable_device_counts()
    tr = LocalTransport(k)
    dt = inp.dt if dt is None else dt
    torch = slabs[0].torch
    with torch.cuda.stream(slabs[0].stream):  # the copies run on the library's stream (one context per device)
        for _ in range(steps):
            for s in slabs:
                s.pack_dev("halo")
            tr.exchange_all_fixed(slabs, "halo")
            for s in slabs:
                s.set_halo_dev()
                s.advance_dev(dt)
                s.pack_dev("mig")
            tr.exchange_all_fixed(slabs, "mig")
            for s in slabs:
                s.take_migrants_dev()
    return assemble([s.owned() for s in slabs], inp.positions.shape[0])


def assemble(parts, n: int):
    """Global (positions, velocities) from every slab's owned atoms."""
    pos, vel = np.full((n, 3), np.nan), np.full((n, 3), np.nan)
    seen = np.zeros(n, np.int64)
    for p, v, g in parts:
        pos[g], vel[g] = p, v
        np.add.at(seen, g, 1)
    if not np.all(seen == 1):
        raise RuntimeError("slab decomposition lost or duplicated atoms")
    return pos, vel

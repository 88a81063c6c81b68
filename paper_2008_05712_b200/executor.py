"""Real-time launch site for combined work requests (north star (1)-(2),
SURVEY.md §8f-1).

The reference drives the BH force phase through its message-driven runtime:
one work request per bucket (buffer_indices = the bucket's walk_order,
hr/workloads/nbody.py:304-316), the occupancy / arrival-gap trigger combines
them (hr/aggregator.py:91-110), the data manager plans the batch
(hr/memory.py:289-360) and ``Timeline._launch_gpu`` charges a COST MODEL for
the transfer and the kernel (hr/timeline.py:300-321).  Here the same API runs
for real on the B200:

  * ``Runtime`` / ``AggregatorState`` / ``poll_combine`` unchanged (host);
    ``max_size`` comes from the occupancy of the real member kernel;
  * the device data manager plans the batch (residency, LRU, min-free-slot,
    per-member address maps -- bit-identical to the reference's plans);
  * ``gc_dm_stage_bh`` moves the missing buffers' payloads (node COM/mass or
    bucket particles) into their HBM slots: the reorganised staging layout;
  * ``gc_bh_run_members`` evaluates every member bucket from its address map
    (one warp per member), and the completion fans out to the owners.

Arrival times are the workload's schedule (the reference's ``_schedule``,
nbody.py:285-301); batches execute on the device as they are emitted and
each batch's device time is recorded, so the combine / reuse experiments
(hr/experiments.py:113-132) run on hardware instead of the cost model.

With ``ewald`` set, every bucket also submits the second kernel class of
NBodyParams(ewald=True) (nbody.py:317-323): buffers [bucket], item_count
max(1, n_b), its own trigger state (max_size from the real ewald member
kernel's occupancy) and its own data manager (the Timeline splits the
capacity per class, hr/timeline.py:153-155); classes are polled in sorted
order (hr/timeline.py:262-266).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .aggregator import AggregatorState, compute_max_size, poll_combine
from .devicesim import b200_device_spec, b200_kernel_spec
from .memory import DeviceMemory, MemoryMode
from .errors import HeteroRtError
from .nbody import DEFAULT_SOFTENING
from .runtime import CompletionEvent, Runtime


@dataclass
class BatchRecord:
    """One combined launch (the reference's ScheduleLog row, hr/timeline.py:63-100)."""
    combined_id: int
    members: int
    positions: int
    transferred: int
    transfer_bytes: int
    indirection_bytes: int
    transactions: int
    emit_time: float
    device_ms: float
    kernel_class: str = "force"


@dataclass
class RunResult:
    forces: np.ndarray
    batches: list = field(default_factory=list)
    wall_s: float = 0.0
    ewald_forces: np.ndarray | None = None  # g m_i a_corr (periodic correction), ewald class only
    ewald_pot: np.ndarray | None = None

    @property
    def device_ms(self) -> float:
        return sum(b.device_ms for b in self.batches)

    @property
    def transfer_bytes(self) -> int:
        return sum(b.transfer_bytes for b in self.batches)


def plan_kinds(ptr, ids, kind, buckets, sorted_members: bool) -> np.ndarray:
    """Kind (0 node, 1 particle interaction) of every position of a combined
    request's plan: the member buckets' lists concatenated, each member in id
    order when the plan sorts it (REUSE_SORTED, hr/memory.py:342-347)."""
    buckets = np.asarray(buckets, np.int64)
    if len(buckets) == 0:
        return np.zeros(0, np.int8)
    lo, hi = ptr[buckets], ptr[buckets + 1]
    ln = hi - lo
    seg = np.repeat(np.arange(len(buckets)), ln)
    pos = np.arange(int(ln.sum())) - np.repeat(np.cumsum(ln) - ln, ln) + np.repeat(lo, ln)
    kd = kind[pos]
    if sorted_members:
        kd = kd[np.lexsort((ids[pos], seg))]
    return np.ascontiguousarray(kd, dtype=np.int8)


class DeviceBatcher:
    """The device batcher of one kernel class (gc_batcher_*, csrc/batcher.cu):
    vectorised submission into a device ring, the trigger of
    hr/aggregator.py:41-110 (observe + poll at every arrival, size rule and
    strict timeout rule), and per emitted batch the device data manager's plan,
    the slot staging and one member-kernel launch -- all asynchronous; the
    host synchronises once in ``log``."""

    def __init__(self, tree, memory: DeviceMemory, max_size: int, timeout_factor: float = 2.0, window: int = 0,
                 g: float = 1.0, eps: float = DEFAULT_SOFTENING):
        self.tree, self.memory = tree, memory
        self._ctx = L.context()
        self.handle = C.c_void_p()
        L.call("gc_batcher_create", self._ctx.handle, tree.handle, memory.handle, int(max_size),
               float(timeout_factor), int(window), float(g), float(eps), C.byref(self.handle))

    def __del__(self):
        try:
            if self.handle:
                L.load().gc_batcher_destroy(self.handle)
        except Exception:
            pass

    def submit(self, owners, arrivals, ptr, ids, kinds) -> None:
        owners, ptr, ids = L.i64(owners), L.i64(ptr), L.i64(ids)
        arrivals = L.f64(arrivals)
        kinds = np.ascontiguousarray(kinds, np.int8)
        L.call("gc_batcher_submit", self.handle, len(owners), L.ptr(owners, L.i64p), L.ptr(arrivals, L.f64p),
               L.ptr(ptr, L.i64p), L.ptr(ids, L.i64p), L.ptr(kinds, L.i8p))

    def submit_walk(self, owners, arrivals) -> None:
        """Requests whose buffers are the owners' device-walk lists (no buffer
        id leaves the device; see gc_batcher_submit_walk)."""
        owners, arrivals = L.i64(owners), L.f64(arrivals)
        L.call("gc_batcher_submit_walk", self.handle, len(owners), L.ptr(owners, L.i64p), L.ptr(arrivals, L.f64p))

    def prepare(self, ptr, max_id: int) -> None:
        """Size every device buffer for a phase of len(ptr) - 1 requests."""
        ptr = L.i64(ptr)
        L.call("gc_batcher_prepare", self.handle, len(ptr) - 1, L.ptr(ptr, L.i64p), int(max_id))

    def poll(self, now: float) -> None:
        L.call("gc_batcher_poll", self.handle, float(now))

    def flush(self, now: float) -> None:
        L.call("gc_batcher_flush", self.handle, float(now))

    def log(self):
        """Synchronise; ScheduleLog rows: int64 (n, 7) {combined_id, first
        request, members, positions, transferred, transactions, synchronous
        plan} and float64 (n, 2) {emit time, device ms}."""
        n = np.zeros(1, np.int64)
        L.call("gc_batcher_sync", self.handle, L.ptr(n, L.i64p))
        rows = np.zeros((int(n[0]), 7), np.int64)
        times = np.zeros((int(n[0]), 2))
        L.call("gc_batcher_log", self.handle, L.ptr(rows, L.i64p), L.ptr(times, L.f64p))
        return rows, times

    @staticmethod
    def trigger_device(max_size: int, timeout_factor: float, window: int, arrivals=None, n: int | None = None,
                       is_poll=None):
        """The trigger alone, evaluated on the device: emissions (first
        request, count, time) for events at `arrivals` (is_poll[i] != 0: a
        poll, else an arrival), or for n arrivals stamped by %globaltimer."""
        if arrivals is not None:
            arrivals = L.f64(arrivals)
            n = len(arrivals)
        ip = None if is_poll is None else np.ascontiguousarray(is_poll, np.int8)
        cap = max(int(n), 1)
        f, c, t = np.zeros(cap, np.int64), np.zeros(cap, np.int64), np.zeros(cap)
        ne = np.zeros(1, np.int64)
        L.call("gc_batcher_trigger_device", int(max_size), float(timeout_factor), int(window), int(n),
               None if arrivals is None else L.ptr(arrivals, L.f64p), None if ip is None else L.ptr(ip, L.i8p),
               L.ptr(f, L.i64p), L.ptr(c, L.i64p),
               L.ptr(t, L.f64p), L.ptr(ne, L.i64p))
        k = int(ne[0])
        return f[:k], c[:k], t[:k]


class GpuForceExecutor:
    """Runs one BH force phase through the runtime API on the device."""

    def __init__(self, tree, lists, mode: MemoryMode = MemoryMode.REUSE_SORTED, capacity_bytes: int = 8 << 20,
                 slot_bytes: int = 256, g: float = 1.0, eps: float = DEFAULT_SOFTENING,
                 timeout_factor: float = 2.0, max_size: int | None = None, ewald=None,
                 ewald_max_size: int | None = None, device_batcher: bool = True):
        self.tree = tree
        self.ptr, self.ids, self.kind, self.item_count = lists.csr()
        self.mode = mode
        self.g, self.eps = g, eps
        self.ewald = ewald
        classes = ["ewald", "force"] if ewald is not None else ["force"]
        per_class = max(slot_bytes, capacity_bytes // len(classes))  # hr/timeline.py:153-155
        self.memories = {c: DeviceMemory(per_class, slot_bytes, mode) for c in classes}
        self.memory = self.memories["force"]
        if max_size is None:
            max_size = compute_max_size(b200_kernel_spec("force_slot"), b200_device_spec())
        self.runtime = Runtime()
        self.states = {"force": AggregatorState("force", int(max_size), timeout_factor)}
        if ewald is not None:
            if tree.dim != 3:
                raise ValueError("the ewald class needs a 3-D tree")
            if ewald_max_size is None:
                ewald_max_size = compute_max_size(b200_kernel_spec("ewald_member"), b200_device_spec())
            self.states["ewald"] = AggregatorState("ewald", int(ewald_max_size), timeout_factor)
            self.bucket_node = np.asarray(tree.bucket_ids, np.int64)
            self.bucket_n = np.asarray(tree._load()["pcount"], np.int64)[self.bucket_node]
        for c in sorted(self.states):
            self.runtime.register_group(self.states[c])
        self.state = self.states["force"]
        self._next_id = 0
        self.plan_log = None  # set to a list to record every plan (host-driven path)
        self.device_batcher = device_batcher  # the force class through gc_batcher (no ewald class, no plan log)
        self.batcher = None
        if device_batcher and ewald is None:  # created and sized with the executor (not in the timed phase)
            st = self.state
            self.batcher = DeviceBatcher(tree, self.memory, st.max_size, st.timeout_factor, st.window, g, eps)
            self.batcher.prepare(self.ptr, int(self.ids.max()) if len(self.ids) else 0)

    # -- one combined launch (replaces Timeline._launch_gpu's cost model) ----------
    def _member_kinds(self, buckets) -> np.ndarray:
        return plan_kinds(self.ptr, self.ids, self.kind, buckets, self.mode is MemoryMode.REUSE_SORTED)

    def launch(self, combined, now: float) -> BatchRecord:
        cls = combined.members[0].kernel_class
        mem = self.memories[cls]
        members = [wr.buffer_indices for wr in combined.members]
        buckets = np.array([wr.owner for wr in combined.members], np.int64)
        plan, layout = mem.build_plan(members, now)
        if self.plan_log is not None:  # parity instrumentation: (class, members, now, transfers, addresses)
            self.plan_log.append((cls, members, now, [b for b, _ in plan.to_transfer], layout.addresses.copy()))
        npos = int(layout.member_bounds[-1])
        L.call("gc_dm_stage_bh", mem.handle, self.tree.handle)
        if cls == "force":
            kinds = self._member_kinds(buckets)
            L.call("gc_bh_run_members", self.tree.handle, mem.handle, L.ptr(L.i64(buckets), L.i64p),
                   len(buckets), L.ptr(kinds, L.i8p), npos, float(self.g), float(self.eps))
        else:
            L.call("gc_bh_run_ewald", self.tree.handle, mem.handle, L.ptr(L.i64(buckets), L.i64p), len(buckets),
                   L.ptr(self.ewald.array(), L.f64p), float(self.g))
        tm = np.zeros(3)
        L.call("gc_bh_timings", self.tree.handle, L.ptr(tm, L.f64p))  # staging + member kernel (events)
        mem.release_batch(members)
        self.runtime.on_completion(CompletionEvent(combined.combined_id, [wr.id for wr in combined.members],
                                                   "gpu", now))
        return BatchRecord(combined.combined_id, len(members), npos, len(plan.to_transfer), plan.total_bytes,
                           plan.indirection_bytes, int(layout.total_transactions()), now, float(tm[0] + tm[1]), cls)

    # -- the force phase through the device batcher -----------------------------------
    def _run_device_batcher(self, times, buckets=None) -> RunResult:
        owners = np.arange(len(self.ptr) - 1) if buckets is None else np.asarray(buckets, np.int64)
        nb = len(owners)
        st = self.state
        res = RunResult(forces=None)
        t0 = time.perf_counter()
        bat = self.batcher  # the prepared batcher serves one phase; a later phase gets a fresh one
        self.batcher = None
        if bat is None:
            bat = DeviceBatcher(self.tree, self.memory, st.max_size, st.timeout_factor, st.window, self.g, self.eps)
        self.runtime.submit_to_device("force", nb)
        try:  # the lists are the tree's device walk: submit them where they are
            bat.submit_walk(owners, times)
        except HeteroRtError as e:
            if type(e) is not HeteroRtError:  # GC_E_STATE only (no device-resident lists): a host submission
                raise
            if buckets is not None:  # the CSR of the listed buckets
                lens = self.ptr[owners + 1] - self.ptr[owners]
                sub = np.concatenate([[0], np.cumsum(lens)])
                pos = np.concatenate([np.arange(self.ptr[b], self.ptr[b + 1]) for b in owners]) if len(owners) \
                    else np.zeros(0, np.int64)
                bat.submit(owners, times, sub, self.ids[pos], self.kind[pos])
            else:
                bat.submit(owners, times, self.ptr, self.ids, self.kind)
        bat.flush(float(times[-1]) if nb else 0.0)  # end of the phase (hr/timeline.py:276-298)
        rows, tms = bat.log()
        res.wall_s = time.perf_counter() - t0
        indirect = self.mode is not MemoryMode.REDUNDANT
        for r, t in zip(rows, tms):
            res.batches.append(BatchRecord(self._next_id, int(r[2]), int(r[3]), int(r[4]),
                                           int(r[4]) * self.memory.slot_bytes, 4 * int(r[3]) if indirect else 0,
                                           int(r[5]), float(t[0]), float(t[1])))
            self._next_id += 1
            self.runtime.complete_on_device(int(r[2]))
        self.last_batcher = bat
        out = np.zeros((self.tree.n, self.tree.dim))
        L.call("gc_bh_get_forces", self.tree.handle, L.ptr(out, L.f64p))
        res.forces = out
        return res

    # -- the force phase ------------------------------------------------------------
    def run(self, arrival_times=None, buckets=None) -> RunResult:
        """One work request per bucket (DFS order) at `arrival_times` (default:
        back to back) -- plus its ewald request when enabled; returns the
        forces and the per-batch log.  `buckets` (device batcher only): the
        requests of these buckets alone (arrival_times per listed bucket)."""
        from .aggregator import make_combined
        nb = len(self.ptr) - 1 if buckets is None else len(buckets)
        times = np.zeros(nb) if arrival_times is None else np.asarray(arrival_times, float)
        if self.device_batcher and self.ewald is None and self.plan_log is None:
            return self._run_device_batcher(times, buckets)
        if buckets is not None:
            raise ValueError("a bucket subset runs through the device batcher only")
        res = RunResult(forces=None)
        t0 = time.perf_counter()
        for b in range(nb):
            ids = self.ids[self.ptr[b]:self.ptr[b + 1]]
            wr = self.runtime.make_work_request(b, "force", ids, int(self.item_count[b]), times[b])
            self.runtime.submit_work_request(wr, times[b])
            if self.ewald is not None:
                node = int(self.bucket_node[b])
                ew = self.runtime.make_work_request(b, "ewald", (node,), max(1, int(self.bucket_n[b])), times[b])
                self.runtime.submit_work_request(ew, times[b])
            for cls in sorted(self.states):  # hr/timeline.py:262-266
                c = poll_combine(self.states[cls], times[b], self._next_id)
                if c is not None:
                    res.batches.append(self.launch(c, times[b]))
                    self._next_id += 1
        # end of the phase: drain in max_size chunks (hr/timeline.py:276-298)
        end = float(times[-1]) if nb else 0.0
        for cls in sorted(self.states):
            st = self.states[cls]
            while st.pending:
                take = [st.pending.popleft() for _ in range(min(st.max_size, len(st.pending)))]
                res.batches.append(self.launch(make_combined(take, end, self._next_id), end))
                self._next_id += 1
        res.wall_s = time.perf_counter() - t0
        out = np.zeros((self.tree.n, self.tree.dim))
        L.call("gc_bh_get_forces", self.tree.handle, L.ptr(out, L.f64p))
        res.forces = out
        if self.ewald is not None:
            f, p = np.zeros((self.tree.n, 3)), np.zeros(self.tree.n)
            L.call("gc_bh_get_ewald", self.tree.handle, L.ptr(f, L.f64p), L.ptr(p, L.f64p))
            res.ewald_forces, res.ewald_pot = f, p
        return res

"""Data-reorganisation-with-reuse layer, device-resident (mirrors hr/memory.py).

Same names and semantics as the reference: ``MemoryMode`` (30-40),
``DeviceSlot`` (43-47), ``ChareTable`` (50-75), ``lookup_residency`` (78-93),
``DeviceHeap`` (96-122), ``SortedIndexArray`` (125-179), ``TransferPlan`` /
``AccessLayout`` / ``transaction_count`` (182-225) and ``DeviceMemory``
(228-369).  The residency table, pin counts, LRU eviction order, slot
allocation and the per-member address maps live in HBM and are computed by
libgcharm's data-manager kernels (csrc/dm.cu); the Python objects here are
views over that state.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib as L
from .errors import CapacityError

HALF_WARP = 16
ADDRESS_BYTES = 4


class MemoryMode(Enum):
    REDUNDANT = "redundant"
    REUSE = "reuse"
    REUSE_SORTED = "reuse_sorted"

    @classmethod
    def parse(cls, name: str) -> "MemoryMode":
        for m in cls:
            if m.value == name:
                return m
        raise ValueError(f"unknown memory mode {name!r}")


_MODE_CODE = {MemoryMode.REDUNDANT: 0, MemoryMode.REUSE: 1, MemoryMode.REUSE_SORTED: 2}


@dataclass
class DeviceSlot:
    slot_index: int
    size_bytes: int
    last_use_time: float


class ChareTable:
    """Snapshot view of the device buffer -> slot map."""

    def __init__(self, mem: "DeviceMemory"):
        self._mem = mem

    def _entries(self) -> dict:
        return self._mem._table()

    def __contains__(self, buffer: int) -> bool:
        return buffer in self._entries()

    def __len__(self) -> int:
        return len(self._entries())

    def get(self, buffer: int):
        return self._entries().get(buffer)

    def buffers(self) -> list:
        return list(self._entries())

    def slot_indices(self) -> list:
        return [s.slot_index for s in self._entries().values()]


def lookup_residency(table, buffer_indices, now: float = 0.0):
    """Partition into (resident, missing), preserving order; residents get
    their LRU timestamp refreshed (hr/memory.py:78-93)."""
    mem = table._mem if isinstance(table, ChareTable) else table
    ids = L.i64(list(buffer_indices))
    res = np.zeros(len(ids), np.int8)
    if len(ids):
        L.call("gc_dm_lookup", mem.handle, L.ptr(ids, L.i64p), len(ids), float(now), L.ptr(res, L.i8p))
    resident = [int(b) for b, r in zip(ids, res) if r]
    missing = [int(b) for b, r in zip(ids, res) if not r]
    return resident, missing


class DeviceHeap:
    """View of the uniform-slot pool (hr/memory.py:96-122)."""

    def __init__(self, mem: "DeviceMemory"):
        self._mem = mem
        self.capacity_bytes = mem.capacity_bytes
        self.slot_bytes = mem.slot_bytes
        self.slot_count = mem.capacity_bytes // mem.slot_bytes

    @property
    def free_slots(self) -> int:
        return int(self._mem._state()[1])

    @property
    def used_bytes(self) -> int:
        return (self.slot_count - self.free_slots) * self.slot_bytes


class SortedIndexArray:
    """Strictly ascending deduplicated indices with a comparison counter
    (hr/memory.py:125-175; host-side instrumentation fed by observe_indices)."""

    def __init__(self):
        self._a: list[int] = []
        self.comparisons = 0
        self.inserts = 0

    def __len__(self):
        return len(self._a)

    @property
    def indices(self):
        return list(self._a)

    def _lower_bound(self, idx: int, count: bool) -> int:
        lo, hi = 0, len(self._a)
        while lo < hi:
            mid = (lo + hi) >> 1
            if count:
                self.comparisons += 1
            if self._a[mid] < idx:
                lo = mid + 1
            else:
                hi = mid
        return lo

    def position(self, idx: int):
        k = self._lower_bound(idx, False)
        return k if k < len(self._a) and self._a[k] == idx else None

    def insert(self, idx: int) -> int:
        self.inserts += 1
        k = self._lower_bound(idx, True)
        if k < len(self._a):
            self.comparisons += 1
            if self._a[k] == idx:
                return k
        self._a.insert(k, idx)
        return k


def insert_sorted_index(arr: SortedIndexArray, idx: int) -> int:
    return arr.insert(idx)


class DeviceSortedIndex:
    """The SortedIndexArray a DeviceMemory observes, held on the device
    (gc_dm_observe / gc_dm_sorted_index): same indices, comparisons and
    inserts as the reference's binary insertion (memory.py:125-179)."""

    def __init__(self, mem: "DeviceMemory"):
        self._mem = mem

    def _state(self, with_indices: bool):
        out = np.zeros(3, np.int64)
        L.call("gc_dm_sorted_index", self._mem.handle, L.ptr(out, L.i64p), None)
        idx = None
        if with_indices:
            idx = np.zeros(int(out[0]), np.int64)
            L.call("gc_dm_sorted_index", self._mem.handle, L.ptr(out, L.i64p), L.ptr(idx, L.i64p))
        return out, idx

    def __len__(self):
        return int(self._state(False)[0][0])

    @property
    def indices(self):
        return self._state(True)[1].tolist()

    @property
    def comparisons(self) -> int:
        return int(self._state(False)[0][1])

    @property
    def inserts(self) -> int:
        return int(self._state(False)[0][2])

    def position(self, idx: int):
        a = self._state(True)[1]
        k = int(np.searchsorted(a, idx))
        return k if k < len(a) and a[k] == idx else None


@dataclass
class TransferPlan:
    to_transfer: list  # (buffer index, bytes)
    total_bytes: int
    indirection_bytes: int
    mode: MemoryMode


@dataclass
class AccessLayout:
    """Device slot address per logical item position, one warp per member."""

    addresses: np.ndarray
    member_bounds: np.ndarray
    indirect: bool
    transactions: np.ndarray | None = None  # per member, computed on device with the plan

    def address_of(self, position: int) -> int:
        return int(self.addresses[position])

    def member_addresses(self, m: int) -> np.ndarray:
        return self.addresses[self.member_bounds[m]: self.member_bounds[m + 1]]

    def member_transactions(self) -> list:
        if self.transactions is not None:
            return [int(x) for x in self.transactions]
        from .kernels import count_address_runs
        mult = 2 if self.indirect else 1
        return [count_address_runs(self.member_addresses(m), HALF_WARP) * mult
                for m in range(len(self.member_bounds) - 1)]

    def total_transactions(self) -> int:
        return sum(self.member_transactions())


def transaction_count(layout: AccessLayout, item_count: int) -> int:
    """hr/memory.py:215-225"""
    from .kernels import count_address_runs
    if item_count < 1:
        raise ValueError("item_count must be >= 1")
    runs = count_address_runs(layout.addresses[:item_count], HALF_WARP)
    return runs * 2 if layout.indirect else runs


class DeviceMemory:
    """Residency manager for one kernel class, state in HBM (gc_dm)."""

    def __init__(self, capacity_bytes: int, slot_bytes: int, mode: MemoryMode):
        if slot_bytes <= 0 or capacity_bytes < slot_bytes:
            raise ValueError("heap needs room for at least one slot")
        self.mode = mode
        self.capacity_bytes = int(capacity_bytes)
        self.slot_bytes = int(slot_bytes)
        self._ctx = L.context()
        self.handle = C.c_void_p()
        L.call("gc_dm_create", self._ctx.handle, self.capacity_bytes, self.slot_bytes, _MODE_CODE[mode],
               C.byref(self.handle))
        self.heap = DeviceHeap(self)
        self.table = ChareTable(self)
        self.sorted_index = DeviceSortedIndex(self)

    def __del__(self):
        try:
            if self.handle:
                L.load().gc_dm_destroy(self.handle)
        except Exception:
            pass

    # -- state views ------------------------------------------------------------
    def _state(self):
        out = np.zeros(4, np.int64)
        L.call("gc_dm_state", self.handle, L.ptr(out, L.i64p))
        return out

    def _table(self) -> dict:
        n = int(self._state()[2])
        bufs, slots, lu, pins = (np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(n), np.zeros(n, np.int64))
        if n:
            L.call("gc_dm_table", self.handle, L.ptr(bufs, L.i64p), L.ptr(slots, L.i64p), L.ptr(lu, L.f64p),
                   L.ptr(pins, L.i64p))
        return {int(b): DeviceSlot(int(s), self.slot_bytes, float(t)) for b, s, t in zip(bufs, slots, lu)}

    # -- pinning -------------------------------------------------------------------
    def pin(self, buffers) -> None:
        ids = L.i64(list(buffers))
        if len(ids):
            L.call("gc_dm_pin", self.handle, L.ptr(ids, L.i64p), len(ids), 1)

    def unpin(self, buffers) -> None:
        ids = L.i64(list(buffers))
        if len(ids):
            L.call("gc_dm_pin", self.handle, L.ptr(ids, L.i64p), len(ids), -1)

    def observe_indices(self, buffer_indices) -> None:
        """Feed request indices into the per-class sorted array in REUSE_SORTED
        mode (hr/memory.py:252-256) -- on the device (gc_dm_observe)."""
        if self.mode is MemoryMode.REUSE_SORTED:
            ids = L.i64(np.asarray(buffer_indices, np.int64).reshape(-1))
            if len(ids):
                L.call("gc_dm_observe", self.handle, L.ptr(ids, L.i64p), len(ids))

    # -- eviction ----------------------------------------------------------------
    def evict_slots(self, needed_bytes: int) -> list:
        out = np.zeros(max(1, self.heap.slot_count), np.int64)
        n = np.zeros(1, np.int64)
        try:
            L.call("gc_dm_evict", self.handle, int(needed_bytes), L.ptr(out, L.i64p), L.ptr(n, L.i64p))
        except CapacityError:
            raise
        return [int(x) for x in out[: int(n[0])]]

    # -- planning ----------------------------------------------------------------
    def build_plan(self, member_indices, now: float = 0.0):
        """hr/memory.py:289-360 on the device; returns (TransferPlan, AccessLayout)."""
        members = [np.asarray(m, dtype=np.int64).reshape(-1) for m in member_indices]
        bounds = np.zeros(len(members) + 1, np.int64)
        bounds[1:] = np.cumsum([len(m) for m in members])
        ids = np.ascontiguousarray(np.concatenate(members)) if bounds[-1] else np.zeros(1, np.int64)
        nt, npos = np.zeros(1, np.int64), np.zeros(1, np.int64)
        L.call("gc_dm_build_plan", self.handle, L.ptr(ids, L.i64p), L.ptr(bounds, L.i64p), len(members),
               float(now), L.ptr(nt, L.i64p), L.ptr(npos, L.i64p))
        tt = np.zeros(max(1, int(nt[0])), np.int64)
        addr = np.zeros(max(1, int(npos[0])), np.int64)
        tx = np.zeros(max(1, len(members)), np.int64)
        ob = np.zeros(3, np.int64)
        L.call("gc_dm_plan_get", self.handle, L.ptr(tt, L.i64p), L.ptr(addr, L.i64p), L.ptr(tx, L.i64p),
               L.ptr(ob, L.i64p))
        plan = TransferPlan(to_transfer=[(int(b), self.slot_bytes) for b in tt[: int(nt[0])]],
                            total_bytes=int(ob[0]), indirection_bytes=int(ob[1]), mode=self.mode)
        layout = AccessLayout(addresses=addr[: int(npos[0])].copy(), member_bounds=bounds, indirect=bool(ob[2]),
                              transactions=tx[: len(members)].copy())
        return plan, layout

    def release_batch(self, member_indices) -> None:
        if self.mode is MemoryMode.REDUNDANT:
            return
        parts = [np.asarray(m, dtype=np.int64).reshape(-1) for m in member_indices]
        ids = np.ascontiguousarray(np.concatenate(parts)) if parts else np.zeros(0, np.int64)
        if len(ids):
            L.call("gc_dm_release", self.handle, L.ptr(ids, L.i64p), len(ids))

    def check_injective(self) -> bool:
        slots = self.table.slot_indices()
        return len(slots) == len(set(slots))

"""Data manager / trigger / partitioner restatements — CPU ORACLE (tests only).

Straight-line Python restatements of the reference's integer decision logic,
written independently of both the reference classes and the product:

* ``OracleDM`` restates ``DeviceMemory`` (hr/memory.py:228-369): residency
  lookup with LRU refresh (78-93), min-free-slot heap (96-122), LRU eviction of
  unpinned buffers keyed by (last_use_time, buffer) (260-285), first-seen
  dedup + optional ascending allocation (319-341), per-member address map,
  sorted per member in REUSE_SORTED (342-347), REDUNDANT staging (302-317) and
  pin counting (240-250, 362-365).
* ``emissions`` restates the combining rule of ``poll_combine`` /
  ``observe_arrival`` (hr/aggregator.py:41-110).
* ``partition`` restates ``partition_queue`` (hr/scheduler.py:73-107).
* ``count_runs`` restates ``count_address_runs`` (hr/kernels.py:168-177).
"""

from __future__ import annotations

import bisect


class OracleCapacityError(Exception):
    pass


class OracleDM:
    def __init__(self, capacity_bytes, slot_bytes, mode):
        if slot_bytes <= 0 or capacity_bytes < slot_bytes:
            raise ValueError("need at least one slot")
        self.mode = mode  # "redundant" | "reuse" | "reuse_sorted"
        self.slot_bytes = slot_bytes
        self.capacity = capacity_bytes
        self.n_slots = capacity_bytes // slot_bytes
        self.free = list(range(self.n_slots))  # kept sorted: smallest first
        self.slot_of = {}
        self.last_use = {}
        self.pins = {}

    # pin counts are per distinct buffer per call
    def _pin(self, bufs):
        for b in set(bufs):
            self.pins[b] = self.pins.get(b, 0) + 1

    def _unpin(self, bufs):
        for b in set(bufs):
            c = self.pins.get(b, 0) - 1
            if c > 0:
                self.pins[b] = c
            else:
                self.pins.pop(b, None)

    def evict(self, needed_bytes):
        if needed_bytes > self.capacity:
            raise OracleCapacityError("exceeds capacity")
        have = len(self.free) * self.slot_bytes
        out = []
        if have >= needed_bytes:
            return out
        order = sorted((self.last_use[b], b) for b in self.slot_of if b not in self.pins)
        for _, b in order:
            if have >= needed_bytes:
                break
            s = self.slot_of.pop(b)
            del self.last_use[b]
            bisect.insort(self.free, s)
            out.append(b)
            have += self.slot_bytes
        if have < needed_bytes:
            raise OracleCapacityError("pinned")
        return out

    def plan(self, members, now=0.0):
        """Returns dict(to_transfer, total_bytes, indirection_bytes, addresses,
        bounds, indirect)."""
        bounds = [0]
        for m in members:
            bounds.append(bounds[-1] + len(m))
        if self.mode == "redundant":
            flat = [b for m in members for b in m]
            if len(flat) > self.n_slots:
                raise OracleCapacityError("staging exceeds slots")
            return dict(to_transfer=flat, total_bytes=len(flat) * self.slot_bytes, indirection_bytes=0,
                        addresses=list(range(len(flat))), bounds=bounds, indirect=False)
        seen, distinct = set(), []
        for m in members:
            for b in m:
                if b not in seen:
                    seen.add(b)
                    distinct.append(b)
        missing = []
        for b in distinct:
            if b in self.slot_of:
                self.last_use[b] = now
            else:
                missing.append(b)
        if self.mode == "reuse_sorted":
            missing.sort()
        self._pin(distinct)
        try:
            self.evict(len(missing) * self.slot_bytes)
        except OracleCapacityError:
            self._unpin(distinct)
            raise
        for b in missing:
            if not self.free:
                raise OracleCapacityError("heap full")
            self.slot_of[b] = self.free.pop(0)
            self.last_use[b] = now
        addresses = []
        for m in members:
            seq = sorted(m) if self.mode == "reuse_sorted" else m
            addresses.extend(self.slot_of[b] for b in seq)
        return dict(to_transfer=missing, total_bytes=len(missing) * self.slot_bytes,
                    indirection_bytes=4 * len(addresses), addresses=addresses, bounds=bounds, indirect=True)

    def release(self, members):
        if self.mode == "redundant":
            return
        self._unpin([b for m in members for b in m])

    def injective(self):
        s = list(self.slot_of.values())
        return len(s) == len(set(s))


def count_runs(addresses, group=16):
    total = 0
    for s in range(0, len(addresses), group):
        chunk = addresses[s: s + group]
        total += 1 + sum(1 for a, b in zip(chunk, chunk[1:]) if b != a + 1)
    return total


def member_transactions(plan, group=16):
    mult = 2 if plan["indirect"] else 1
    a, bd = plan["addresses"], plan["bounds"]
    return [count_runs(a[bd[i]: bd[i + 1]], group) * mult for i in range(len(bd) - 1)]


def emissions(arrivals, max_size, poll_times, timeout_factor=2.0):
    """Combined batches emitted by the trigger for (time, id) arrivals polled at
    the union of poll and arrival times; [(time, (ids...)), ...]."""
    out, pend = [], []
    last, maxgap = None, None
    times = sorted(set(poll_times) | {t for t, _ in arrivals})
    k = 0
    for now in times:
        while k < len(arrivals) and arrivals[k][0] <= now:
            t, i = arrivals[k]
            if last is not None:
                g = t - last
                maxgap = g if maxgap is None or g > maxgap else maxgap
            last = t
            pend.append(i)
            k += 1
        while len(pend) >= max_size:
            out.append((now, tuple(pend[:max_size])))
            del pend[:max_size]
        if pend and maxgap is not None and now - last > timeout_factor * maxgap:
            out.append((now, tuple(pend)))
            pend = []
    return out


def partition(items, share, nearest_target=False):
    """Prefix split by cumulative item count; returns the cut index."""
    total = sum(items)
    target = total * share
    if not items or target <= 0.0:
        return 0
    cum = 0.0
    for i, w in enumerate(items):
        cum += w
        if cum >= target:
            if nearest_target and (cum - target) > (target - (cum - w)):
                return i
            return i + 1
    return len(items)

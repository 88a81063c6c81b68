"""Work-request stream capture and replay (mirrors hr/workloads/trace.py).

A trace is line-delimited text, one work request per line
(hr/workloads/trace.py:1-9, 22-62):

    arrival_time kernel_class idx0,idx1,... item_count bytes_per_item

with ``repr`` floats so a dump / parse round trip is exact.  Here a trace is
also the fixture feed of the B200 batcher: a recorded BH
force stream is replayed through the device executor (``replay_forces``) --
trigger, device data manager, slot staging, member kernel -- without
re-running the walk that produced it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import TraceFormatError


@dataclass(frozen=True)
class TraceRecord:
    arrival_time: float
    kernel_class: str
    buffer_indices: tuple
    item_count: int
    bytes_per_item: int

    def to_line(self) -> str:
        idx = ",".join(str(int(i)) for i in self.buffer_indices)
        return f"{self.arrival_time!r} {self.kernel_class} {idx} {self.item_count} {self.bytes_per_item}"


def dump_trace(records, path) -> None:
    Path(path).write_text("".join(r.to_line() + "\n" for r in records))


def parse_trace(path) -> list:
    """hr/workloads/trace.py:43-62: 5 fields, >= 1 item and >= 1 buffer."""
    records = []
    for line_no, raw in enumerate(Path(path).read_text().splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) != 5:
            raise TraceFormatError(line_no, f"expected 5 fields, got {len(parts)}")
        try:
            t = float(parts[0])
            indices = tuple(int(x) for x in parts[2].split(","))
            items = int(parts[3])
            bpi = int(parts[4])
        except ValueError as exc:
            raise TraceFormatError(line_no, str(exc)) from None
        if items < 1 or not indices:
            raise TraceFormatError(line_no, "need at least one item and one buffer")
        records.append(TraceRecord(t, parts[1], indices, items, bpi))
    return records


def trace_roundtrip(records, path) -> list:
    """Dump, re-parse and diff (hr/workloads/trace.py:65-76); [] = faithful."""
    dump_trace(records, path)
    back = parse_trace(path)
    problems = []
    if len(back) != len(records):
        problems.append(f"length {len(records)} -> {len(back)}")
    for i, (a, b) in enumerate(zip(records, back)):
        if a != b:
            problems.append(f"line {i + 1}: {a} != {b}")
    return problems


def nbody_schedule(item_counts, seed: int = 42, pieces: int = 16, emit_cost: float = 1e-4,
                   piece_gap: float = 4.0) -> list:
    """Walk-ordered arrival times of the BH force requests (NBodyWorkload._schedule,
    hr/workloads/nbody.py:285-301): dense inside a tree piece, lognormal lulls
    between pieces."""
    rng = np.random.default_rng(seed + 1)
    n = len(item_counts)
    per_piece = max(1, math.ceil(n / pieces))
    times, t = [], 0.0
    for i, ic in enumerate(item_counts):
        if i > 0 and i % per_piece == 0:
            t += piece_gap * float(rng.lognormal(mean=0.0, sigma=1.0))
        t += emit_cost * max(1, int(ic))
        times.append(t)
    return times


def nbody_stream(ptr, ids, item_count, seed: int = 42, pieces: int = 16, emit_cost: float = 1e-4,
                 piece_gap: float = 4.0, bytes_per_item: int = 48) -> list:
    """One "force" record per bucket (DFS order): buffers = its walk_order
    (hr/workloads/trace.py:80-97 without the Ewald class)."""
    times = nbody_schedule(item_count, seed, pieces, emit_cost, piece_gap)
    return [TraceRecord(t, "force", tuple(int(x) for x in ids[ptr[b]:ptr[b + 1]]), int(item_count[b]),
                        bytes_per_item) for b, t in enumerate(times)]


def replay_forces(records, tree, lists, **executor_kw):
    """Replay a recorded BH force stream on the device: the k-th "force" record
    is bucket k's request (streams are emitted in DFS bucket order); its
    buffers must equal that bucket's device-walk list.  Returns the executor's
    RunResult (forces + per-batch log)."""
    from .executor import GpuForceExecutor
    force = [r for r in records if r.kernel_class == "force"]
    ex = GpuForceExecutor(tree, lists, **executor_kw)
    if len(force) != len(ex.ptr) - 1:
        raise ValueError(f"trace has {len(force)} force records for {len(ex.ptr) - 1} buckets")
    for b, r in enumerate(force):
        if not np.array_equal(np.asarray(r.buffer_indices, np.int64), ex.ids[ex.ptr[b]:ex.ptr[b + 1]]):
            raise ValueError(f"trace record {b} does not match bucket {b}'s interaction list")
        if r.item_count != int(ex.item_count[b]):
            raise ValueError(f"trace record {b}: item_count {r.item_count} != {int(ex.item_count[b])}")
    return ex.run([r.arrival_time for r in force])


# -- large streams (SURVEY.md §8f-2 at configs[2] / configs[3] scale) ------------
# A text trace of the 1M-particle BH force phase would hold ~10^8 buffer ids
# (hundreds of MB of text); the same records are kept in a compact binary
# form: arrival times, the buffer CSR (ptr, ids), kinds and item counts.

def dump_stream_npz(path, times, ptr, ids, item_count, kinds, buckets=None) -> None:
    """One "force" record per bucket k (or per bucket buckets[k]): arrival
    times[k], buffers ids[ptr[k]:ptr[k+1]] with kinds (0 node, 1 particle
    interaction), item_count[k] -- the content of the text trace lines, binary."""
    extra = {} if buckets is None else {"buckets": np.asarray(buckets, np.int64)}
    np.savez(path, times=np.asarray(times, np.float64), ptr=np.asarray(ptr, np.int64),
             ids=np.asarray(ids, np.int32), kinds=np.asarray(kinds, np.int8),
             item_count=np.asarray(item_count, np.int64), **extra)


def load_stream_npz(path) -> dict:
    z = np.load(path)
    s = {k: z[k] for k in ("times", "ptr", "ids", "kinds", "item_count")}
    if "buckets" in z:
        s["buckets"] = z["buckets"]
    n = len(s["times"])
    if len(s["ptr"]) != n + 1 or len(s["item_count"]) != n or s["ptr"][-1] != len(s["ids"]):
        raise TraceFormatError(0, "inconsistent stream arrays")
    if np.any(np.diff(s["times"]) < 0):
        raise TraceFormatError(0, "arrival times decrease")
    return s


def replay_stream(stream: dict, tree, lists, **executor_kw):
    """Replay a binary force stream on the device batcher (the requests must
    be the tree's buckets in DFS order with their device-walk lists)."""
    from .executor import GpuForceExecutor
    ex = GpuForceExecutor(tree, lists, **executor_kw)
    b = stream.get("buckets")
    if b is None:
        if len(stream["times"]) != len(ex.ptr) - 1:
            raise ValueError(f"stream has {len(stream['times'])} records for {len(ex.ptr) - 1} buckets")
        if not (np.array_equal(stream["ptr"], ex.ptr) and np.array_equal(stream["ids"], ex.ids)
                and np.array_equal(stream["kinds"], ex.kind) and np.array_equal(stream["item_count"], ex.item_count)):
            raise ValueError("stream records do not match the tree's interaction lists")
        return ex.run(stream["times"])
    # a sampled stream: the records of buckets b (configs[3] scale)
    lens = ex.ptr[b + 1] - ex.ptr[b]
    if not (np.array_equal(np.diff(stream["ptr"]), lens) and np.array_equal(stream["item_count"], ex.item_count[b])):
        raise ValueError("stream records do not match the tree's interaction lists")
    pos = np.concatenate([np.arange(ex.ptr[x], ex.ptr[x + 1]) for x in b]) if len(b) else np.zeros(0, np.int64)
    if not (np.array_equal(stream["ids"], ex.ids[pos]) and np.array_equal(stream["kinds"], ex.kind[pos])):
        raise ValueError("stream records do not match the tree's interaction lists")
    return ex.run(stream["times"], buckets=b)

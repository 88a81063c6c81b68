"""Host-side runtime pieces: trigger, occupancy model, runtime, partitioners.

Pinned against the reference's emissions/partitions (tests/golden) and its
unit fixtures (pkg/tests/test_aggregator.py, test_devicesim.py,
test_runtime.py, test_scheduler.py).  No GPU needed.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import dm as odm
from paper_2008_05712_b200 import aggregator as agg
from paper_2008_05712_b200 import devicesim as ds
from paper_2008_05712_b200 import scheduler as sch
from paper_2008_05712_b200.errors import (ClockError, ConsistencyError, DuplicateWorkRequestError, GroupingError,
                                          KernelFitError, MeasurementError, RoutingError)
from paper_2008_05712_b200.runtime import CompletionEvent, Message, Runtime, WorkRequest


def wr(i, cls="force", buffers=(0,), items=1, t=0.0):
    return WorkRequest(i, 0, cls, list(buffers), items, t)


def test_max_size_presets():
    k20 = ds.DEVICE_PRESETS["kepler-k20"]
    assert agg.compute_max_size(ds.KERNEL_PRESETS["force"], k20) == 104
    assert agg.compute_max_size(ds.KERNEL_PRESETS["ewald"], k20) == 65
    assert agg.compute_max_size(ds.KernelSpec("k", 128, 1, 1, 1.0), ds.DeviceSpec(1, 128, 1, 1 << 16, 1 << 16)) == 1
    b, occ = ds.calc_occupancy(ds.KERNEL_PRESETS["force"], k20)
    assert b == 8 and occ == 0.5


def test_occupancy_matches_oracle():
    rng = np.random.default_rng(2024)
    for _ in range(3000):
        d = ds.DeviceSpec(int(rng.integers(1, 32)), int(rng.integers(128, 4096)), int(rng.integers(1, 33)),
                          int(rng.integers(1 << 12, 1 << 17)), int(rng.integers(1 << 12, 1 << 17)))
        k = ds.KernelSpec("r", int(rng.integers(1, 1025)), int(rng.integers(1, 256)), int(rng.integers(1, 1 << 15)))
        try:
            b, _ = ds.calc_occupancy(k, d)
        except KernelFitError:
            b = 0
        assert b == ds.occupancy_oracle(k, d)


def test_observe_arrival_rules():
    s = agg.AggregatorState("force", max_size=104)
    for t in (0.0, 5.0, 7.0):
        agg.observe_arrival(s, t)
    assert s.max_interval == 5.0
    s = agg.AggregatorState("force", max_size=104, window=2)
    for t in (0.0, 10.0, 11.0, 12.0):
        agg.observe_arrival(s, t)
    assert s.max_interval == 1.0
    with pytest.raises(ClockError):
        agg.observe_arrival(s, 1.0)
    with pytest.raises(GroupingError):
        agg.make_combined([wr(0), wr(1, "ewald")], 0.0)
    with pytest.raises(GroupingError):
        agg.make_combined([], 0.0)


def test_emissions_match_reference_golden():
    g = json.load(open(os.path.join(GOLDEN, "aggregator.json")))
    for e in g["emissions"]:
        arrivals = [tuple(a) for a in e["arrivals"]]
        state = agg.AggregatorState("force", max_size=e["max_size"])
        got, ai = [], 0
        for pt in sorted(set(e["polls"]) | {a for a, _ in arrivals}):
            while ai < len(arrivals) and arrivals[ai][0] <= pt:
                at, aid = arrivals[ai]
                state.pending.append(wr(aid, t=at))
                agg.observe_arrival(state, at)
                ai += 1
            while True:
                b = agg.poll_combine(state, pt)
                if b is None:
                    break
                got.append([pt, [m.id for m in b.members]])
        assert got == e["emissions"]


def test_static_count():
    s = agg.StaticCountAggregation(3)
    assert [s.on_arrival() for _ in range(7)] == [False, False, True, False, False, True, False]


def test_partition_queue_golden_and_kway_k2():
    g = json.load(open(os.path.join(GOLDEN, "aggregator.json")))
    for p in g["partitions"]:
        q = [wr(i, items=w) for i, w in enumerate(p["items"])]
        part = sch.partition_queue(q, sch.PerfEstimate(), cpu_share=p["share"], nearest_target=p["nearest"])
        assert len(part.cpu_set) == p["cut"]
        b = sch.partition_k(p["items"], [p["share"], 1.0 - p["share"]], p["nearest"])
        if p["share"] * sum(p["items"]) > 0:
            assert b[1] == p["cut"]


def test_kway_partition_properties():
    rng = np.random.default_rng(7)
    for _ in range(200):
        k = int(rng.integers(1, 9))
        w = [int(x) for x in rng.integers(1, 100, size=int(rng.integers(1, 300)))]
        est = sch.KWayEstimate(k)
        for d in range(k):
            est.record(d, 100, float(rng.uniform(0.5, 2.0)))
        b = sch.partition_k(w, est.shares())
        assert b[0] == 0 and b[-1] == len(w) and all(x <= y for x, y in zip(b, b[1:]))
    # equal speeds: near-equal item shares
    w = [1] * 1000
    b = sch.partition_k(w, [0.25] * 4)
    assert b == [0, 250, 500, 750, 1000]


def test_perf_estimate():
    est = sch.PerfEstimate()
    assert sch.current_ratio(est) == (0.5, 0.5)
    sch.record_sample(est, sch.CPU, 10, 1.0)
    sch.record_sample(est, sch.GPU, 10, 0.25)
    c, g = sch.current_ratio(est)
    assert abs(c - 0.2) < 1e-12 and abs(g - 0.8) < 1e-12
    with pytest.raises(MeasurementError):
        sch.record_sample(est, sch.GPU, 0, 1.0)
    assert odm.partition([10, 20, 30, 40], 0.6) == 3  # prefix crossing (test_scheduler.py:73-78)
    part = sch.partition_queue([wr(i, items=x) for i, x in enumerate([10, 20, 30, 40])], est, cpu_share=0.6)
    assert [w.item_count for w in part.cpu_set] == [10, 20, 30]


def test_runtime_semantics():
    rt = Runtime()
    hits = []
    a = rt.create_chare({"go": (2, lambda ctx, m: hits.append(m.target))})
    assert rt.dispatch_ready(Message(a, "go")) is None
    assert rt.dispatch_ready(Message(a, "go")) is not None
    assert hits == [a]
    with pytest.raises(RoutingError):
        rt.dispatch_ready(Message(99, "go"))
    rt.register_group(agg.AggregatorState("force", 4))
    w0 = rt.make_work_request(a, "force", [1, 2], 3, 0.0)
    rt.submit_work_request(w0, 0.0)
    with pytest.raises(DuplicateWorkRequestError):
        rt.submit_work_request(w0, 0.0)
    with pytest.raises(RoutingError):
        rt.submit_work_request(rt.make_work_request(a, "md", [1], 1, 0.0), 0.0)
    msgs = rt.on_completion(CompletionEvent(0, [w0.id], "GPU", 1.0))
    assert len(msgs) == 1 and msgs[0].entry_method == "work_done"
    with pytest.raises(ConsistencyError):
        rt.on_completion(CompletionEvent(0, [w0.id], "GPU", 1.0))
    assert rt.pending_count == 0 and rt.completed_count == 1

"""Device batcher (csrc/batcher.cu, executor.DeviceBatcher):
the trigger of hr/aggregator.py on the device against the reference's
recorded emissions and the host poll_combine, and whole force phases through
the batcher against the host-driven launch path (same batches, same plans'
transfer and transaction counts, bit-identical forces) and the oracle."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

FORCE_RTOL = 1e-5


def test_device_trigger_matches_reference_emissions():
    """gc_batcher_trigger_device on the golden traces (hr/aggregator.py
    emissions recorded by tests/golden/make_golden.py): arrivals plus the
    timeline's extra polls, same batches at the same times."""
    from paper_2008_05712_b200.executor import DeviceBatcher
    g = json.load(open(os.path.join(GOLDEN, "aggregator.json")))
    for e in g["emissions"]:
        arr = [tuple(a) for a in e["arrivals"]]
        assert [i for _, i in arr] == list(range(len(arr)))
        times, poll = [], []
        k = 0
        for now in sorted(set(e["polls"]) | {t for t, _ in arr}):  # arrivals at `now` first, then a poll
            while k < len(arr) and arr[k][0] <= now:
                times.append(arr[k][0])
                poll.append(0)
                k += 1
            times.append(now)
            poll.append(1)
        f, c, t = DeviceBatcher.trigger_device(e["max_size"], 2.0, 0, np.array(times), is_poll=np.array(poll))
        got = [[float(tt), list(range(int(ff), int(ff + cc)))] for ff, cc, tt in zip(f, c, t)]
        assert got == e["emissions"]


@pytest.mark.parametrize("window", [0, 1, 3])
def test_device_trigger_matches_poll_combine(window):
    """Random bursty traces: the device trigger equals the Python
    observe_arrival / poll_combine (hr/aggregator.py mirror) polled after
    every arrival, with and without a gap window; %globaltimer stamps give a
    FIFO partition of all arrivals."""
    from paper_2008_05712_b200.aggregator import AggregatorState, observe_arrival, poll_combine
    from paper_2008_05712_b200.executor import DeviceBatcher
    from paper_2008_05712_b200.runtime import WorkRequest
    rng = np.random.default_rng(7 + window)
    for trial in range(5):
        n = int(rng.integers(50, 400))
        gaps = np.where(rng.random(n) < 0.1, rng.uniform(2, 8, n), rng.uniform(0, 0.5, n))
        t = np.cumsum(gaps)
        ms = int(rng.integers(1, 40))
        st = AggregatorState("force", ms, 2.0, window=window)
        ref = []
        for i in range(n):
            st.pending.append(WorkRequest(i, 0, "force", [], 1, t[i], 0))
            observe_arrival(st, t[i])
            while (c := poll_combine(st, t[i])) is not None:
                ref.append((c.members[0].id, len(c.members), t[i]))
        f, c, tt = DeviceBatcher.trigger_device(ms, 2.0, window, t)
        assert [(int(a), int(b), float(x)) for a, b, x in zip(f, c, tt)] == ref
    f, c, tt = DeviceBatcher.trigger_device(16, 2.0, 0, None, n=1000)  # real time: %globaltimer stamps
    assert np.all(np.diff(tt) >= 0) and np.array_equal(f, np.concatenate([[0], np.cumsum(c)[:-1]]))
    assert c.sum() <= 1000 and np.all(c <= 16)


@pytest.fixture(scope="module")
def problem():
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.fp32_exact(gen.gen_particles(6000, 11, clustering=0.6, dim=3))
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, 0.6, ps)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    ol = orc.build_interaction_lists(ot, 0.6)
    ref = orc.eval_forces(ot, ol, ps.positions, ps.masses)
    return ps, tree, lists, ref


@pytest.mark.parametrize("mode,cap,max_size,bursty", [("redundant", 64 << 20, 64, False),
                                                      ("reuse", 4 << 20, 64, False),
                                                      ("reuse_sorted", 4 << 20, 64, True),
                                                      ("reuse_sorted", 1500 * 256, 48, True),
                                                      ("reuse", 1500 * 256, 48, False)])
def test_batcher_equals_host_path(problem, mode, cap, max_size, bursty):
    """The batcher path and the host-driven path (device_batcher=False) emit
    the same batches and their plans transfer the same buffers with the same
    transaction counts; forces are bit-identical and within 1e-5 of the
    oracle.  A 1500-slot heap makes plans evict (the synchronous fallback)."""
    from paper_2008_05712_b200.executor import GpuForceExecutor
    from paper_2008_05712_b200.memory import MemoryMode
    ps, tree, lists, ref = problem
    nb = len(lists.csr()[0]) - 1
    t = None
    if bursty:
        rng = np.random.default_rng(3)
        t = np.cumsum(np.where(np.arange(nb) % 40 == 0, 5.0, 0.01) * rng.uniform(0.5, 1.5, nb))
    runs = []
    for dev in (True, False):
        ex = GpuForceExecutor(tree, lists, MemoryMode.parse(mode), capacity_bytes=cap, slot_bytes=256,
                              max_size=max_size, device_batcher=dev)
        r = ex.run(t)
        assert ex.runtime.completed_count == nb and ex.runtime.pending_count == 0
        runs.append(r)
    a, b = runs
    assert [x.members for x in a.batches] == [x.members for x in b.batches]
    assert [x.positions for x in a.batches] == [x.positions for x in b.batches]
    assert [x.transferred for x in a.batches] == [x.transferred for x in b.batches]
    assert [x.transactions for x in a.batches] == [x.transactions for x in b.batches]
    assert [x.emit_time for x in a.batches] == [x.emit_time for x in b.batches]
    np.testing.assert_array_equal(a.forces, b.forces)
    err = np.linalg.norm(a.forces - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= FORCE_RTOL


def test_batcher_config1_scale():
    """configs[0] (Plummer 16K, theta 0.7) through the batcher in the three
    memory modes: every request completes once, transfers equal the host path."""
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    from paper_2008_05712_b200.executor import GpuForceExecutor
    from paper_2008_05712_b200.memory import MemoryMode
    ps = gen.fp32_exact(gen.gen_plummer(16384, 42))
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, 0.7, ps)
    for mode in ("redundant", "reuse", "reuse_sorted"):
        cap = 1 << 30 if mode == "redundant" else 64 << 20
        rs = [GpuForceExecutor(tree, lists, MemoryMode.parse(mode), capacity_bytes=cap, slot_bytes=256,
                               device_batcher=d).run() for d in (True, False)]
        assert [x.transferred for x in rs[0].batches] == [x.transferred for x in rs[1].batches]
        assert [x.transactions for x in rs[0].batches] == [x.transactions for x in rs[1].batches]
        np.testing.assert_array_equal(rs[0].forces, rs[1].forces)

"""The reference's recorded BH force stream replayed on the device batcher
(trace.replay_forces -> executor): forces within 1e-5 of the oracle."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_replay_reference_trace():
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody, trace
    from paper_2008_05712_b200.memory import MemoryMode
    recs = trace.parse_trace(os.path.join(GOLDEN, "trace_nbody3d_1500.txt"))
    ps = gen.gen_particles(1500, 5, clustering=0.6, dim=3)
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, 0.6, ps)
    res = trace.replay_forces(recs, tree, lists, mode=MemoryMode.REUSE_SORTED, capacity_bytes=1 << 20, max_size=40)
    # the reference's particles are not float32-representable: evaluate the
    # reference lists at the float32-rounded inputs the device computes with
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    r32 = gen.fp32_exact(ps)
    ref = orc.eval_forces(ot, orc.build_interaction_lists(ot, 0.6), r32.positions, r32.masses)
    err = np.linalg.norm(res.forces - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= 1e-5
    assert len(res.batches) > len(recs) // 40  # the recorded lulls trigger timeout flushes


def test_replay_1m_stream(tmp_path):
    """configs[2] at full size (clustered 1M, theta 0.7): the force phase's
    work-request stream (one request per bucket, arrivals from the workload's
    schedule, hr/workloads/nbody.py:285-301) dumped once, reloaded and
    replayed through the device batcher -- trigger, device data manager with
    reuse, staging, member kernel -- forces within 1e-5 of the union path."""
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody, trace
    from paper_2008_05712_b200.memory import MemoryMode
    ps = gen.fp32_exact(gen.gen_particles(1_000_000, 42, clustering=0.6, dim=3))
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, 0.7, ps)
    ref = nbody.eval_forces(tree, lists, ps)
    ptr, ids, kind, ic = lists.csr()
    times = trace.nbody_schedule(ic, seed=42)
    path = tmp_path / "stream_1m.npz"
    trace.dump_stream_npz(path, times, ptr, ids, ic, kind)
    s = trace.load_stream_npz(path)
    res = trace.replay_stream(s, tree, lists, mode=MemoryMode.REUSE_SORTED, capacity_bytes=256 << 20)
    assert sum(b.members for b in res.batches) == len(ic)
    assert len(res.batches) >= len(ic) // max(b.members for b in res.batches)
    err = np.linalg.norm(res.forces - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= 1e-5
    assert sum(b.transferred for b in res.batches) < len(ids)  # reuse: far fewer transfers than references


def test_replay_16m_stream_sample(tmp_path):
    """configs[3]'s system (Plummer 2^24) on one GPU: the work-request stream
    of a 3,000-walk-group sample of buckets (the device walk over that range,
    gc_bh_set_range) dumped, reloaded and replayed through the device batcher
    (reuse-sorted data manager sized for every node id: asynchronous plans);
    the sampled buckets' forces within 1e-5 of the union path.  (The full
    16M stream would hold ~2.7e9 buffer ids: sampled.)"""
    import ctypes as C

    from paper_2008_05712_b200 import _lib as L
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody, trace
    from paper_2008_05712_b200.memory import MemoryMode
    ps = gen.fp32_exact(gen.gen_plummer(1 << 24, 42))
    tree = nbody.build_bucket_tree(ps, 8)
    nwg = C.c_int64()
    L.call("gc_bh_groups", tree.handle, C.byref(nwg), None)
    first = np.zeros(nwg.value + 1, np.int64)
    L.call("gc_bh_groups", tree.handle, C.byref(nwg), L.ptr(first, L.i64p))
    g0 = nwg.value // 2
    g1 = g0 + 3000
    L.call("gc_bh_set_range", tree.handle, g0, g1)
    lists = nbody.build_interaction_lists(tree, 0.7, ps)
    ref = nbody.eval_forces(tree, lists, ps)
    ptr, ids, kind, ic = lists.csr()
    b = np.arange(first[g0], first[g1])
    lens = ptr[b + 1] - ptr[b]
    sub = np.concatenate([[0], np.cumsum(lens)])
    pos = np.concatenate([np.arange(ptr[x], ptr[x + 1]) for x in b])
    times = trace.nbody_schedule(ic[b], seed=42)
    path = tmp_path / "stream_16m_sample.npz"
    trace.dump_stream_npz(path, times, sub, ids[pos], ic[b], kind[pos], buckets=b)
    s = trace.load_stream_npz(path)
    cap = (int(tree.sizes()[0]) + 1) * 256
    res = trace.replay_stream(s, tree, lists, mode=MemoryMode.REUSE_SORTED, capacity_bytes=cap)
    assert sum(x.members for x in res.batches) == len(b)
    nodes = np.asarray(tree.bucket_ids)[b]
    ps0, pc = np.asarray(tree.pstart)[nodes], np.asarray(tree.pcount)[nodes]
    parts = np.asarray(tree.pidx)[np.repeat(ps0, pc) + np.arange(pc.sum()) - np.repeat(np.cumsum(pc) - pc, pc)]
    err = np.linalg.norm(res.forces[parts] - ref[parts], axis=1) / np.linalg.norm(ref[parts], axis=1)
    assert len(parts) > 100_000 and err.max() <= 1e-5

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

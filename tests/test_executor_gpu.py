"""Combined work requests on the device through the reference's runtime API
(executor.py): trigger -> device data manager plan -> slot staging -> member
kernel.  Forces must match the oracle's eval_forces (<= 1e-5 per particle,
FP32 path) in every memory mode, with evictions, and every work request must
complete exactly once."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FORCE_RTOL = 1e-5


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


def rel_err(a, b):
    return np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)


@pytest.mark.parametrize("mode", ["redundant", "reuse", "reuse_sorted"])
def test_executor_matches_oracle(problem, mode):
    from paper_2008_05712_b200.executor import GpuForceExecutor
    from paper_2008_05712_b200.memory import MemoryMode
    ps, tree, lists, ref = problem
    cap = (64 << 20) if mode == "redundant" else (4 << 20)
    ex = GpuForceExecutor(tree, lists, MemoryMode.parse(mode), capacity_bytes=cap, slot_bytes=256, max_size=64)
    res = ex.run()
    nb = len(ex.ptr) - 1
    assert ex.runtime.completed_count == nb and ex.runtime.pending_count == 0
    assert sum(b.members for b in res.batches) == nb
    assert rel_err(res.forces, ref).max() <= FORCE_RTOL
    if mode != "redundant":
        assert ex.memory.check_injective()


def test_executor_evictions_and_timeouts(problem):
    """A small heap forces LRU evictions; a bursty schedule triggers timeout flushes."""
    from paper_2008_05712_b200.executor import GpuForceExecutor
    from paper_2008_05712_b200.memory import MemoryMode
    ps, tree, lists, ref = problem
    ex = GpuForceExecutor(tree, lists, MemoryMode.REUSE_SORTED, capacity_bytes=1500 * 256, slot_bytes=256,
                          max_size=48)
    nb = len(ex.ptr) - 1
    rng = np.random.default_rng(3)
    t = np.cumsum(np.where(np.arange(nb) % 40 == 0, 5.0, 0.01) * rng.uniform(0.5, 1.5, nb))
    res = ex.run(t)
    assert rel_err(res.forces, ref).max() <= FORCE_RTOL
    sizes = [b.members for b in res.batches]
    assert max(sizes) <= 48 and min(sizes) < 48  # size-rule and timeout flushes both occurred
    assert ex.runtime.completed_count == nb


@pytest.mark.parametrize("mode,cap,max_size", [("redundant", 1 << 30, None), ("reuse", 64 << 20, None),
                                               ("reuse_sorted", 64 << 20, None), ("reuse", 1 << 19, 64),
                                               ("reuse_sorted", 1 << 19, 64)])
def test_config1_runtime_path_plans_match_oracle(mode, cap, max_size):
    """configs[0] at the runtime path's own scale (Plummer 16K, theta 0.7,
    one request per bucket, max_size from the real member kernel's
    occupancy, or 64 with a 512 KiB heap to force LRU evictions): every
    device plan -- transfers in order, address maps -- equals the oracle data
    manager (oracle/dm.py, pinned to hr/memory.py); forces within 1e-5."""
    from oracle import dm as odm
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    from paper_2008_05712_b200.executor import GpuForceExecutor
    from paper_2008_05712_b200.memory import MemoryMode
    ps = gen.fp32_exact(gen.gen_plummer(16384, 42))
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, 0.7, ps)
    ex = GpuForceExecutor(tree, lists, MemoryMode.parse(mode), capacity_bytes=cap, slot_bytes=256,
                          max_size=max_size)
    ex.plan_log = []
    res = ex.run()
    assert len(ex.plan_log) == len(res.batches) >= 1
    if max_size:
        assert len(res.batches) >= 5730 // 64
    ora = odm.OracleDM(cap, 256, mode)
    for cls, members, now, transfers, addresses in ex.plan_log:
        q = ora.plan(members, now=now)
        assert transfers == q["to_transfer"]
        assert addresses.tolist() == q["addresses"]
        ora.release(members)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    ref = orc.eval_forces(ot, orc.build_interaction_lists(ot, 0.7), ps.positions, ps.masses)
    assert rel_err(res.forces, ref).max() <= FORCE_RTOL

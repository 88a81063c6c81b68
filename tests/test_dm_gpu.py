"""GPU parity of the device data manager against the reference's plans.

Bar: bit-exact to_transfer order, slot addresses, member bounds, byte counts,
transaction counts, residency table and CapacityError behaviour
(hr/memory.py:228-369; golden plans from tests/golden/make_golden.py, plus the
reference's own unit fixtures, pkg/tests/test_memory.py:85-273).
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import dm as odm

pytestmark = pytest.mark.gpu

MODES = {"redundant": "REDUNDANT", "reuse": "REUSE", "reuse_sorted": "REUSE_SORTED"}


@pytest.fixture(scope="module")
def mm():
    from paper_2008_05712_b200 import memory
    return memory


def test_golden_plans(mm):
    from paper_2008_05712_b200.errors import CapacityError
    cases = json.load(open(os.path.join(GOLDEN, "dm_plans.json")))
    for c in cases:
        mem = mm.DeviceMemory(c["cap"], c["slot"], mm.MemoryMode[MODES[c["mode"]]])
        for (members, now), want in zip(c["batches"], c["result"]):
            try:
                plan, layout = mem.build_plan(members, now)
            except CapacityError:
                assert not want["ok"], c["name"]
                continue
            assert want["ok"], c["name"]
            assert [b for b, _ in plan.to_transfer] == want["to_transfer"], c["name"]
            assert layout.addresses.tolist() == want["addresses"], c["name"]
            assert layout.member_bounds.tolist() == want["bounds"]
            assert plan.total_bytes == want["total_bytes"]
            assert plan.indirection_bytes == want["indirection_bytes"]
            assert layout.indirect == want["indirect"]
            assert layout.member_transactions() == want["transactions"], c["name"]
            if c["mode"] != "redundant":
                tab = sorted((b, s.slot_index) for b, s in mem.table._entries().items())
                assert tab == [tuple(x) for x in want["table"]], c["name"]
            if c["release"]:
                mem.release_batch(members)


def test_figure1_fixture(mm):
    for mode, addr, tx in [("REDUNDANT", [0, 1, 2, 3, 4], 1), ("REUSE", [0, 3, 1, 2, 4], 8),
                           ("REUSE_SORTED", [0, 3, 1, 2, 4], 8)]:
        mem = mm.DeviceMemory(1 << 16, 256, mm.MemoryMode[mode])
        if mode != "REDUNDANT":
            mem.build_plan([[2, 5, 7]], now=0.0)
            mem.release_batch([[2, 5, 7]])
        req = [7, 3, 2, 8, 5] if mode == "REUSE_SORTED" else [2, 3, 5, 7, 8]
        plan, layout = mem.build_plan([req], now=1.0)
        assert layout.addresses.tolist() == addr
        assert mm.transaction_count(layout, 5) == tx
        if mode == "REUSE":
            assert [b for b, _ in plan.to_transfer] == [3, 8]
            assert plan.indirection_bytes == 20


def test_eviction_rules(mm):
    from paper_2008_05712_b200.errors import CapacityError
    mem = mm.DeviceMemory(2 * 64, 64, mm.MemoryMode.REUSE)
    for b, t in [(10, 0.0), (11, 1.0), (10, 2.0)]:
        mem.build_plan([[b]], now=t)
        mem.release_batch([[b]])
    assert mem.evict_slots(64) == [11]  # LRU (test_memory.py:164-173)
    mem = mm.DeviceMemory(4 * 64, 64, mm.MemoryMode.REUSE)
    mem.build_plan([[1]], now=0.0)
    mem.release_batch([[1]])
    assert mem.evict_slots(64) == []
    mem = mm.DeviceMemory(2 * 64, 64, mm.MemoryMode.REUSE)
    mem.build_plan([[1, 2]], now=0.0)  # still pinned
    with pytest.raises(CapacityError):
        mem.build_plan([[3]], now=1.0)
    with pytest.raises(CapacityError):
        mem.evict_slots(64 * 3)
    mem = mm.DeviceMemory(2 * 64, 64, mm.MemoryMode.REUSE)
    mem.build_plan([[1, 2]], now=0.0)
    mem.release_batch([[1, 2]])
    mem.build_plan([[3]], now=1.0)  # evicts buffer 1, reuses slot 0
    assert mem.table.get(3).slot_index == 0
    assert 1 not in mem.table


def test_random_interleaving_matches_oracle(mm):
    """plan / release / evict interleavings (test_memory.py:251-273) against the
    straight-line oracle: identical decisions and an injective table."""
    from paper_2008_05712_b200.errors import CapacityError
    rng = np.random.default_rng(33)
    for mode in ("reuse", "reuse_sorted"):
        mem = mm.DeviceMemory(64 * 32, 64, mm.MemoryMode[MODES[mode]])
        ora = odm.OracleDM(64 * 32, 64, mode)
        live = []
        for step in range(300):
            op = rng.integers(0, 3)
            if op == 0 and live:
                batch = live.pop(int(rng.integers(0, len(live))))
                mem.release_batch([batch])
                ora.release([batch])
            elif op == 1:
                need = 64 * int(rng.integers(0, 4))
                try:
                    a, ea = mem.evict_slots(need), None
                except CapacityError:
                    a, ea = None, "cap"
                try:
                    b, eb = ora.evict(need), None
                except odm.OracleCapacityError:
                    b, eb = None, "cap"
                assert ea == eb
                if ea is None:
                    assert a == b
            else:
                req = [int(x) for x in rng.integers(0, 200, size=rng.integers(1, 6))]
                req = list(dict.fromkeys(req))
                try:
                    p, lay = mem.build_plan([req], now=float(step))
                    ok = True
                except CapacityError:
                    ok = False
                try:
                    q = ora.plan([req], now=float(step))
                    ok2 = True
                except odm.OracleCapacityError:
                    ok2 = False
                assert ok == ok2
                if ok:
                    assert [b for b, _ in p.to_transfer] == q["to_transfer"]
                    assert lay.addresses.tolist() == q["addresses"]
                    live.append(req)
            assert mem.check_injective()
            got = sorted((b, s.slot_index) for b, s in mem.table._entries().items())
            assert got == sorted(ora.slot_of.items())


def test_interaction_list_batches_match_oracle(mm):
    """Batches of bucket interaction lists (the force class's real buffer
    streams, 2048 clustered, theta 0.7) through all three modes."""
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    ps = gen.fp32_exact(gen.gen_particles(2048, 12, 0.6, 3))
    t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    L = orc.build_interaction_lists(t, 0.7)
    members = [L.walk_order(b).tolist() for b in range(len(t.buckets))]
    for mode in ("redundant", "reuse", "reuse_sorted"):
        cap = 1 << 24
        mem = mm.DeviceMemory(cap, 256, mm.MemoryMode[MODES[mode]])
        ora = odm.OracleDM(cap, 256, mode)
        for i in range(0, len(members), 104):
            batch = members[i: i + 104]
            p, lay = mem.build_plan(batch, now=float(i))
            q = ora.plan(batch, now=float(i))
            assert [b for b, _ in p.to_transfer] == q["to_transfer"]
            assert lay.addresses.tolist() == q["addresses"]
            assert lay.member_transactions() == odm.member_transactions(q)
            mem.release_batch(batch)
            ora.release(batch)

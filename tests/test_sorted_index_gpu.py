"""SortedIndexArray on the device (hr/memory.py:125-179, fed by
observe_indices 252-256): the sorted distinct set, the comparison count of
the reference's binary insertion and the insert count equal the host
restatement (memory.SortedIndexArray, pinned to the reference's tests in
tests/test_memory_cpu.py) on random chunked streams."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,universe,chunks", [(0, 50, [1, 5, 7, 40]), (1, 5000, [3000, 10, 7000]),
                                                   (2, 300000, [200000, 150000, 1]), (3, 1, [5, 5])])
def test_device_sorted_index_matches_reference(seed, universe, chunks):
    from paper_2008_05712_b200.memory import DeviceMemory, MemoryMode, SortedIndexArray
    rng = np.random.default_rng(seed)
    mem = DeviceMemory(1 << 20, 256, MemoryMode.REUSE_SORTED)
    host = SortedIndexArray()
    for c in chunks:
        ids = rng.integers(0, universe, c)
        mem.observe_indices(ids)
        for b in ids.tolist():
            host.insert(b)
        assert mem.sorted_index.comparisons == host.comparisons
        assert mem.sorted_index.inserts == host.inserts
    assert mem.sorted_index.indices == host.indices
    assert len(mem.sorted_index) == len(host)
    k = host.indices[len(host) // 2]
    assert mem.sorted_index.position(k) == host.position(k)


def test_other_modes_do_not_observe():
    from paper_2008_05712_b200.memory import DeviceMemory, MemoryMode
    mem = DeviceMemory(1 << 20, 256, MemoryMode.REUSE)
    mem.observe_indices([3, 1, 2])
    assert mem.sorted_index.inserts == 0 and len(mem.sorted_index) == 0

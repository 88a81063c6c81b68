"""Host-side pieces of the data-manager mirror that need no GPU."""
import math

import numpy as np

from paper_2008_05712_b200.memory import MemoryMode, SortedIndexArray, insert_sorted_index


def test_sorted_index_array():
    arr = SortedIndexArray()
    for v in [1, 3, 8]:
        arr.insert(v)
    assert insert_sorted_index(arr, 5) == 2
    assert arr.indices == [1, 3, 5, 8]
    assert arr.insert(3) == 1
    assert arr.position(4) is None and arr.position(5) == 2


def test_sorted_index_comparison_bound():
    """pkg/tests/test_acceptance.py:172-193: comparisons <= 2 log2(N!)"""
    rng = np.random.default_rng(404)
    for n in (10, 100, 2000):
        arr = SortedIndexArray()
        vals = rng.integers(0, max(2, n // 2), size=n)
        for v in vals:
            arr.insert(int(v))
        assert arr.indices == sorted(set(vals.tolist()))
        assert arr.comparisons <= max(2.0 * math.lgamma(n + 1) / math.log(2.0), 2.0)


def test_mode_parse():
    assert MemoryMode.parse("reuse_sorted") is MemoryMode.REUSE_SORTED

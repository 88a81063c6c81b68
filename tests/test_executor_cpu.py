"""Host logic of the device batch executor (executor.py): the per-position
kinds of a combined request's plan in list order and in the per-member id
order of REUSE_SORTED plans (hr/memory.py:342-347)."""
import numpy as np

from paper_2008_05712_b200.executor import plan_kinds


def _loop(ptr, ids, kind, buckets, sorted_members):
    out = []
    for b in buckets:
        i, k = ids[ptr[b]:ptr[b + 1]], kind[ptr[b]:ptr[b + 1]]
        if sorted_members:
            k = k[np.argsort(i, kind="stable")]
        out.extend(k.tolist())
    return np.array(out, np.int8)


def test_plan_kinds_matches_loop():
    rng = np.random.default_rng(0)
    nb = 200
    lens = rng.integers(0, 30, nb)
    ptr = np.concatenate([[0], np.cumsum(lens)])
    ids = np.concatenate([rng.choice(5000, size=l, replace=False) for l in lens]).astype(np.int64)
    kind = rng.integers(0, 2, ptr[-1]).astype(np.int8)
    for buckets in ([3, 17, 18, 150], list(range(nb)), [], [199, 0, 42]):
        for s in (False, True):
            np.testing.assert_array_equal(plan_kinds(ptr, ids, kind, buckets, s), _loop(ptr, ids, kind, buckets, s))

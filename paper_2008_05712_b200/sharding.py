"""Sharding the Barnes-Hut force path over the GPUs of one box.

Buckets are independent work units (one chare per bucket,
hr/workloads/nbody.py:305-309).  Every rank holds the particle set and the
tree; the depth-first sequence of walk groups is cut into contiguous ranges
weighted by measured work (n_b * item_count_b) with the K-way generalisation
of ``partition_queue`` (scheduler.partition_k); each rank walks and evaluates
only its range.  Per-GPU times feed ``KWayEstimate`` so later steps shift the
cuts towards faster devices.  There is no collective on the data path; the
force rows of each shard can be assembled with ``allgather_forces`` (NCCL on
GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np

from . import scheduler as sch


def walk_group_weights(wg_first_bucket: np.ndarray, bucket_work: np.ndarray) -> np.ndarray:
    """Work per walk group from per-bucket work."""
    cs = np.concatenate([[0], np.cumsum(bucket_work, dtype=np.int64)])
    return cs[wg_first_bucket[1:]] - cs[wg_first_bucket[:-1]]


def shard_bounds(weights, shares) -> list:
    """K+1 walk-group boundaries for the given device shares."""
    return sch.partition_k([int(w) for w in weights], list(shares))


def shard_tree(tree, rank: int, world: int, estimate: sch.KWayEstimate | None = None):
    """Restrict a device tree (nbody.BucketTree after one full walk) to this
    rank's share of the walk groups; returns (wg_begin, wg_end)."""
    from . import _lib as L
    n = np.zeros(1, np.int64)
    L.call("gc_bh_groups", tree.handle, L.ptr(n, L.i64p), None)
    first = np.zeros(int(n[0]) + 1, np.int64)
    L.call("gc_bh_groups", tree.handle, L.ptr(n, L.i64p), L.ptr(first, L.i64p))
    work = np.zeros(len(tree.bucket_ids), np.int64)
    L.call("gc_bh_bucket_work", tree.handle, L.ptr(work, L.i64p))
    shares = (estimate or sch.KWayEstimate(world)).shares()
    b = shard_bounds(walk_group_weights(first, work), shares)
    L.call("gc_bh_set_range", tree.handle, int(b[rank]), int(b[rank + 1]))
    return int(b[rank]), int(b[rank + 1])


def shard_particles(tree, wg_range) -> np.ndarray:
    """Original particle ids evaluated by a walk-group range."""
    from . import _lib as L
    n = np.zeros(1, np.int64)
    L.call("gc_bh_groups", tree.handle, L.ptr(n, L.i64p), None)
    first = np.zeros(int(n[0]) + 1, np.int64)
    L.call("gc_bh_groups", tree.handle, L.ptr(n, L.i64p), L.ptr(first, L.i64p))
    b0, b1 = first[wg_range[0]], first[wg_range[1]]
    counts = tree.pcount[tree.bucket_ids]
    starts = np.concatenate([[0], np.cumsum(counts)])
    return tree.pidx[starts[b0]: starts[b1]]


def allgather_forces(local_ids: np.ndarray, local_forces: np.ndarray, n: int, group=None) -> np.ndarray:
    """Assemble the full (n, dim) force array from every rank's rows."""
    import torch
    import torch.distributed as dist
    dim = local_forces.shape[1]
    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    cnt = torch.tensor([len(local_ids)], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    m = int(max(c.item() for c in cnts))
    ids = torch.full((m,), -1, dtype=torch.int64, device=dev)
    ids[: len(local_ids)] = torch.as_tensor(local_ids, dtype=torch.int64)
    f = torch.zeros((m, dim), dtype=torch.float64, device=dev)
    f[: len(local_ids)] = torch.as_tensor(local_forces[local_ids], dtype=torch.float64)
    all_ids = [torch.empty_like(ids) for _ in range(world)]
    all_f = [torch.empty_like(f) for _ in range(world)]
    dist.all_gather(all_ids, ids, group=group)
    dist.all_gather(all_f, f, group=group)
    out = np.zeros((n, dim))
    for i, ff in zip(all_ids, all_f):
        i = i.cpu().numpy()
        keep = i >= 0
        out[i[keep]] = ff.cpu().numpy()[keep]
    return out

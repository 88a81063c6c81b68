"""Multi-GPU sharding of the BH path.

CPU (gloo, world_size 2): the host-side shard plan (K-way partition of walk
groups by work) and the force assembly collective, with the float64 oracle
standing in for each rank's device kernels.  GPU: two shards evaluated on one
device reproduce the unsharded forces bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2008_05712_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    ps = gen.fp32_exact(gen.gen_particles(3000, 5, 0.6, 3))
    t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    L = orc.build_interaction_lists(t, 0.7)
    return ps, t, L


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import oracle as orc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ps, t, L = _problem()
        nb = len(t.buckets)
        first = np.arange(0, nb + 32, 32)
        first[-1] = nb
        first = np.unique(first)
        work = t.pcount[t.buckets] * L.item_count
        w = sharding.walk_group_weights(first, work)
        b = sharding.shard_bounds(w, [1.0 / world] * world)
        b0, b1 = int(first[b[rank]]), int(first[b[rank + 1]])
        f_local = orc.eval_forces(t, L, ps.positions, ps.masses, bucket_range=(b0, b1))
        starts = np.concatenate([[0], np.cumsum(t.pcount[t.buckets])])
        ids = t.pidx[starts[b0]: starts[b1]]
        full = sharding.allgather_forces(ids, f_local, len(ps.masses))
        if rank == 0:
            ref = orc.eval_forces(t, L, ps.positions, ps.masses)
            q.put((bool(np.array_equal(full, ref)), b, int(w.sum())))
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_reassemble_exactly():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    ok, bounds, total = q.get(timeout=5)
    assert ok
    assert bounds[0] == 0 and bounds[1] > 0


@pytest.mark.gpu
def test_device_shards_equal_unsharded():
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.fp32_exact(gen.gen_particles(50000, 9, 0.6, 3))
    full_t = nbody.build_bucket_tree(ps, 8)
    full = nbody.eval_forces(full_t, nbody.build_interaction_lists(full_t, 0.7), ps)
    out = np.full_like(full, np.nan)
    for rank in range(2):
        t = nbody.build_bucket_tree(ps, 8)
        nbody.build_interaction_lists(t, 0.7, ps)  # measure work
        rng = sharding.shard_tree(t, rank, 2)
        f = nbody.eval_forces(t, nbody.build_interaction_lists(t, 0.7, ps), ps)
        ids = sharding.shard_particles(t, rng)
        out[ids] = f[ids]
    assert not np.isnan(out).any()
    np.testing.assert_array_equal(out, full)

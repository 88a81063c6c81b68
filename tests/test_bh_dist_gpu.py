"""Distributed Barnes-Hut on the device (bh_dist.py with libgcharm.so):
2 and 3 ranks sharing cuda:0 over gloo (the NCCL path on a multi-GPU box is
the same protocol with device tensors).  Bars: each rank's interaction lists
equal the single-GPU tree's lists for the same buckets, as (level, key
prefix, kind); forces within 1e-5 of the float64 oracle; every particle is
owned by exactly one rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, n, seed, cl, theta):
    import torch.distributed as dist
    from paper_2008_05712_b200 import bh_dist
    from paper_2008_05712_b200 import generators as gen
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ps = gen.fp32_exact(gen.gen_particles(n, seed, clustering=cl, dim=3))
        mine = np.arange(rank, n, world)
        d = bh_dist.DistBH(bh_dist.Comm(), bucket_size=8, theta=theta)
        res = d.step(ps.positions[mine], ps.masses[mine], mine, want_lists=True)
        t = res.tree
        ob = t["buckets"][res.own[0]:res.own[1]]
        q.put((rank, res.gid, res.forces, bh_dist.lists_by_prefix(t, res.lists, res.own),
               bh_dist._key16(t["level"][ob], t["p1"][ob], t["p2"][ob]), res.stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,seed,cl,theta", [(2, 200_000, 42, 0.6, 0.7), (3, 60_000, 9, 0.8, 0.5)])
def test_dist_bh_device_matches_single_gpu(world, n, seed, cl, theta):
    from oracle import oracle as orc
    from paper_2008_05712_b200 import bh_dist
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n, seed, cl, theta)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ps = gen.fp32_exact(gen.gen_particles(n, seed, clustering=cl, dim=3))
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, theta, ps)
    ptr, ids, kind, ic = lists.csr()
    a = tree._load()
    lvl, p1, p2 = bh_dist._node_prefixes(dict(center=a["center"], half=a["half"], first_child=a["first_child"],
                                                n_child=a["n_child"]))
    gb = tree.bucket_ids
    key_g = bh_dist._key16(lvl[gb], p1[gb], p2[gb])
    pos_g = {k: i for i, k in enumerate(key_g.tolist())}
    gtree = dict(level=lvl, p1=p1, p2=p2)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    ref = orc.eval_forces(ot, orc.build_interaction_lists(ot, theta), ps.positions, ps.masses)
    seen = np.zeros(n, np.int64)
    for rank, gid, f, ml, own_keys, stats in out:
        idx = np.array([pos_g[k] for k in own_keys.tolist()])
        assert np.all(np.diff(idx) == 1)
        rl = bh_dist.lists_by_prefix(gtree, (ptr, ids, kind), (int(idx[0]), int(idx[-1]) + 1))
        for x, y in zip(ml, rl):
            np.testing.assert_array_equal(x, y)
        err = np.linalg.norm(f - ref[gid], axis=1) / np.linalg.norm(ref[gid], axis=1)
        assert err.max() <= 1e-5, f"rank {rank}: max rel force err {err.max():.2e}"
        seen[gid] += 1
        print(rank, stats)
    assert np.all(seen == 1)

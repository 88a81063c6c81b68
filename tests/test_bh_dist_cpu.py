"""Distributed Barnes-Hut (bh_dist.py): partitioned trees + LET
exchange over gloo on CPU, world sizes 2 and 3.  The per-rank device work is
replaced by the float64 oracle backend (oracle/dist_backend.py); the protocol
(sample sort, straddling cubes, branch summaries, LET, assembly) is the
product's.  Bars: every rank's interaction lists equal the single-process
reference tree's lists for the same buckets (compared as (level, key prefix,
kind) -- node ids differ between the trees), and its float64 forces are
bit-identical to the single-process oracle forces."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(n, seed, cl):
    from paper_2008_05712_b200 import generators as gen
    return gen.fp32_exact(gen.gen_particles(n, seed, clustering=cl, dim=3))


def _worker(rank, world, port, q, n, seed, cl, theta, shares=None):
    import torch.distributed as dist
    from oracle import oracle as orc
    from oracle.dist_backend import OracleBackend
    from paper_2008_05712_b200 import bh_dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ps = _problem(n, seed, cl)
        mine = np.arange(rank, n, world)  # an arbitrary initial share
        d = bh_dist.DistBH(bh_dist.Comm(), bucket_size=8, theta=theta, backend=OracleBackend(), shares=shares)
        res = d.step(ps.positions[mine], ps.masses[mine], mine, want_lists=True)
        # the single-process reference tree and lists
        gt = orc.build_bucket_tree(ps.positions, ps.masses, 8)
        gl = orc.build_interaction_lists(gt, theta)
        gf = orc.eval_forces(gt, gl, ps.positions, ps.masses)
        gd = dict(center=gt.center, half=gt.half, first_child=gt.first_child, n_child=gt.n_child)
        lvl, p1, p2 = bh_dist._node_prefixes(gd)
        gtree = dict(level=lvl, p1=p1, p2=p2)
        # own buckets of this rank = the global buckets whose particles it holds
        t = res.tree
        ob = t["buckets"][res.own[0]:res.own[1]]
        key_own = bh_dist._key16(t["level"][ob], t["p1"][ob], t["p2"][ob])
        gb = gt.buckets
        key_g = bh_dist._key16(lvl[gb], p1[gb], p2[gb])
        pos_g = {k: i for i, k in enumerate(key_g.tolist())}
        idx = np.array([pos_g[k] for k in key_own.tolist()])
        ok_contig = bool(np.all(np.diff(idx) == 1))
        mine_l = bh_dist.lists_by_prefix(t, res.lists, res.own)
        ref_l = bh_dist.lists_by_prefix(gtree, (gl.ptr, gl.ids, gl.kind), (int(idx[0]), int(idx[-1]) + 1))
        lists_eq = all(np.array_equal(a, b) for a, b in zip(mine_l, ref_l))
        forces_eq = bool(np.array_equal(res.forces, gf[res.gid]))
        q.put((rank, ok_contig, lists_eq, forces_eq, len(res.gid), res.stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,seed,cl,theta", [(2, 6000, 3, 0.6, 0.7), (3, 5000, 11, 0.8, 0.5),
                                                   (2, 3000, 7, 0.0, 0.9)])
def test_dist_bh_lists_and_forces_match_single_process(world, n, seed, cl, theta):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, n, seed, cl, theta)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(o[4] for o in out) == n  # every particle owned by exactly one rank
    for rank, contig, lists_eq, forces_eq, nloc, stats in sorted(out):
        assert contig, f"rank {rank}: own buckets not a contiguous DFS range of the global tree"
        assert lists_eq, f"rank {rank}: lists differ from the single-process tree"
        assert forces_eq, f"rank {rank}: forces differ"
        assert stats["let_nodes_received"] > 0


def test_dist_bh_uneven_shares_move_the_boundary_not_the_results():
    """The balancer's shares (hr/scheduler.py's adaptive split over the
    ranks, scheduler.KWayEstimate) only move the partition: with shares
    0.3 / 0.7 rank 0 owns ~30 % of the particles and every list and float64
    force still equals the single-process reference."""
    world, n = 2, 6000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, n, 3, 0.6, 0.7, [0.3, 0.7])) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(o[4] for o in out) == n
    assert 0.2 * n < out[0][4] < 0.4 * n, [o[4] for o in out]
    for rank, contig, lists_eq, forces_eq, nloc, stats in out:
        assert contig and lists_eq and forces_eq, rank


def test_balancer_shares_follow_speed():
    """KWayEstimate as the distributed step feeds it: equal shares until every
    rank reported, then shares proportional to particles per millisecond."""
    from paper_2008_05712_b200 import scheduler as sch
    b = sch.KWayEstimate(2)
    assert b.shares() == [0.5, 0.5]
    b.record(0, 1000, 2.0)  # 500 particles / ms
    assert b.shares() == [0.5, 0.5]
    b.record(1, 1000, 1.0)  # 1000 particles / ms
    assert np.allclose(b.shares(), [1 / 3, 2 / 3])


def test_key_restatement_orders_like_the_tree():
    """Sorting by the restated octant keys gives the reference tree's
    depth-first particle order (buckets are contiguous key ranges)."""
    from oracle import oracle as orc
    ps = _problem(4000, 5, 0.6)
    k1, k2 = orc.octant_keys(ps.positions, 1.0)
    o = np.lexsort((np.arange(4000), k2, k1))
    t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    at = 0
    for b in t.buckets:  # each bucket = the next contiguous run of the key order
        ids = t.particle_idx(b)
        np.testing.assert_array_equal(np.sort(o[at: at + len(ids)]), ids)
        at += len(ids)
    assert at == 4000

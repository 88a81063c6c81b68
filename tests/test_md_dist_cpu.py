"""Host side of the multi-GPU MD (x-slab decomposition) on CPU:
slab partition, halo / migrant plane selection and the neighbour exchange
protocol over gloo (world sizes 2 and 3, variable message sizes incl. 0)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2008_05712_b200 import md_dist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_bounds_and_neighbours():
    assert md_dist.slab_bounds(24, 5) == [0, 4, 9, 14, 19, 24]
    assert md_dist.slab_bounds(20, 1) == [0, 20]
    with pytest.raises(ValueError):
        md_dist.slab_bounds(3, 4)
    assert md_dist.neighbours(0, 4) == (3, 1)
    assert md_dist.neighbours(3, 4) == (2, 0)
    x = np.array([-1e-9, 0.0, 2.49, 2.5, 59.99, 60.0, 70.0])
    np.testing.assert_array_equal(md_dist.global_cell_x(x, 2.5, 24), [0, 0, 0, 1, 23, 23, 23])


def _planes(x, cell, gnx, bounds, r):
    """Ids of rank r's first / last owned plane (what it sends left / right)."""
    cx = md_dist.global_cell_x(x, cell, gnx)
    return np.nonzero(cx == bounds[r])[0], np.nonzero(cx == bounds[r + 1] - 1)[0]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2008_05712_b200.generators import gen_lj_fcc
        inp = gen_lj_fcc(6, repeat_x=2 * world)
        gnx = inp.cells_xyz[0]
        b = md_dist.slab_bounds(gnx, world)
        tr = md_dist.DistTransport()
        x = inp.positions[:, 0]
        # halo: records = (x, y, z, id) of the first / last owned plane
        sl, sr = _planes(x, inp.cell_size, gnx, b, rank)

        def rec(ids):
            return torch.tensor(np.column_stack([inp.positions[ids], ids]), dtype=torch.float64)

        fl, fr = tr.exchange(rec(sl), rec(sr))
        left, right = md_dist.neighbours(rank, world)
        exp_l = _planes(x, inp.cell_size, gnx, b, left)[1]  # left neighbour's last plane
        exp_r = _planes(x, inp.cell_size, gnx, b, right)[0]
        ok = np.array_equal(fl[:, 3].numpy().astype(np.int64), exp_l) and \
            np.array_equal(fr[:, 3].numpy().astype(np.int64), exp_r) and \
            np.array_equal(fl[:, :3].numpy(), inp.positions[exp_l])
        # migrants: variable sizes including empty messages, 8 words per record
        n_l, n_r = rank % 2, 3 * rank + 1
        ml = torch.full((n_l, 8), float(rank))
        mr = torch.full((n_r, 8), float(rank) + 0.5)
        gl, gr = tr.exchange(ml.double(), mr.double())
        ok = ok and gl.shape == (3 * left + 1, 8) and bool((gl == left + 0.5).all())
        ok = ok and gr.shape == (right % 2, 8) and bool((gr == right).all())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_neighbour_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def _worker_fixed(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = md_dist.DistTransport()
        cap = 16
        left, right = md_dist.neighbours(rank, world)
        n_l, n_r = rank % 3, 2 * rank + 1  # variable fill of fixed-capacity buffers
        send_l = torch.zeros((cap, 4), dtype=torch.float64)
        send_r = torch.zeros((cap, 4), dtype=torch.float64)
        send_l[:n_l] = rank
        send_r[:n_r] = rank + 0.5
        cnt = torch.tensor([n_l, n_r, -1, -1], dtype=torch.int32)
        recv_l = torch.zeros((cap, 4), dtype=torch.float64)
        recv_r = torch.zeros((cap, 4), dtype=torch.float64)
        tr.exchange_fixed(send_l, cnt[0:1], send_r, cnt[1:2], recv_l, cnt[2:3], recv_r, cnt[3:4])
        ok = int(cnt[2]) == 2 * left + 1 and int(cnt[3]) == right % 3
        ok = ok and bool((recv_l[:int(cnt[2])] == left + 0.5).all()) and bool((recv_r[:int(cnt[3])] == right).all())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fixed_capacity_exchange_gloo(world):
    """The device-count step's exchange (fixed-capacity buffers, int32 counts
    sent alongside) over a real process group (gloo on CPU tensors)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_fixed, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res

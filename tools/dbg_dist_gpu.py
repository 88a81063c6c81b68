"""Debug run of the distributed BH on one GPU (gloo ranks sharing cuda:0)."""
import faulthandler
import os
import sys

import numpy as np
import torch.multiprocessing as mp

sys.path.insert(0, ".")


def w(rank, world, port, n):
    faulthandler.enable()
    import torch.distributed as dist
    from paper_2008_05712_b200 import bh_dist
    from paper_2008_05712_b200 import generators as gen
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
    mine = np.arange(rank, n, world)
    d = bh_dist.DistBH(bh_dist.Comm(), bucket_size=8, theta=0.7)
    print(rank, "start", flush=True)
    res = d.step(ps.positions[mine], ps.masses[mine], mine, want_lists=True)
    print(rank, "done", res.stats, np.isfinite(res.forces).all(), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    world, n = int(sys.argv[1]), int(sys.argv[2])
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=w, args=(r, world, 29700 + world, n)) for r in range(world)]
    [p.start() for p in ps]
    [p.join() for p in ps]
    print("exit codes", [p.exitcode for p in ps])

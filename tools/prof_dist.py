"""Host-side profile of one DistBH.step (device backend, gloo, 2 ranks on one GPU): cProfile of rank 0."""
import cProfile
import io
import os
import pstats
import sys

import numpy as np
import torch.multiprocessing as mp

sys.path.insert(0, os.getcwd())


def worker(rank, world, port, n):
    import torch.distributed as dist
    from paper_2008_05712_b200 import bh_dist
    from paper_2008_05712_b200 import generators as gen
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
    mine = np.arange(rank, n, world)
    d = bh_dist.DistBH(bh_dist.Comm(), bucket_size=8, theta=0.7)
    d.step(ps.positions[mine], ps.masses[mine], mine)  # warm-up
    pr = cProfile.Profile()
    pr.enable()
    d.step(ps.positions[mine], ps.masses[mine], mine)
    pr.disable()
    if rank == 0:
        print({k: round(v, 3) for k, v in d.stats.items() if k.startswith('t_')}, flush=True)
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats('tottime').print_stats(25)
        print(s.getvalue()[:6000], flush=True)
    dist.destroy_process_group()


if __name__ == '__main__':
    mp.spawn(worker, args=(2, 29633, int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000), nprocs=2)

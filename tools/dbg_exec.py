import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2008_05712_b200 import generators as gen, nbody, _lib as L
from paper_2008_05712_b200.executor import GpuForceExecutor
from paper_2008_05712_b200.memory import MemoryMode
ps = gen.fp32_exact(gen.gen_plummer(16384, 42))
tree = nbody.build_bucket_tree(ps, 8)
lists = nbody.build_interaction_lists(tree, 0.7, ps)
for mode in ("reuse", "reuse_sorted", "reuse", "reuse_sorted"):
    ex = GpuForceExecutor(tree, lists, MemoryMode.parse(mode), capacity_bytes=64 << 20, slot_bytes=256)
    orig = ex.launch
    def timed(c, now, ex=ex, orig=orig):
        t0 = time.perf_counter(); r = orig(c, now); t1 = time.perf_counter()
        print(f"  {mode} batch {c.combined_id}: members {r.members} pos {r.positions} dev {r.device_ms:.3f} ms wall {1e3*(t1-t0):.1f} ms")
        return r
    ex.launch = timed
    r = ex.run()
    print(mode, "total dev", r.device_ms, "wall", r.wall_s)

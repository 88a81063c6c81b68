"""configs[3] on ONE B200: Plummer 16M, theta 0.7 -- device build, walk, reorg, force timings and memory."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2008_05712_b200 import _lib as L  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402
from paper_2008_05712_b200 import nbody  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
t0 = time.time()
ps = gen.fp32_exact(gen.gen_plummer(n, 42))
print(f"generated {n} in {time.time() - t0:.1f} s", flush=True)
tree = nbody.build_bucket_tree(ps, 8)
ctx = L.context()
tm = np.zeros(3)
w, f, r = [], [], []
for i in range(6):
    L.call("gc_bh_walk", tree.handle, 0.7)
    L.call("gc_bh_forces_async", tree.handle, 1.0, 1e-4)
    L.call("gc_bh_timings", tree.handle, L.ptr(tm, L.f64p))
    if i >= 1:
        w.append(tm[0]); f.append(tm[1]); r.append(tm[2])
inter = nbody.interactions(tree)
sz = tree.sizes()
free, total = torch.cuda.mem_get_info()
fm = statistics.median(f)
step = statistics.median(w) + statistics.median(r) + fm
print(f"n {n}: nodes {sz[0]} buckets {sz[1]} union {sz[3]} records {sz[4]} interactions {inter}")
print(f"walk {statistics.median(w):.3f} ms  reorg {statistics.median(r):.3f} ms  force {fm:.3f} ms  step {step:.3f} ms  "
      f"{inter / step / 1e-3:.3e} interactions/s  force {20 * inter / fm / 1e9:.2f} TFLOP/s  "
      f"device memory used {(total - free) / 2**30:.1f} GiB")

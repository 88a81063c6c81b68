"""Device times of the BH walk and force kernels (CUDA events inside libgcharm), 1M clustered."""
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2008_05712_b200 import _lib as L  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402
from paper_2008_05712_b200 import nbody  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1_000_000
ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
tree = nbody.build_bucket_tree(ps, 8)
ctx = L.context()
staged = "staged" in sys.argv
L.call("gc_bh_set_force_mode", tree.handle, 0 if staged else 1)
tm = np.zeros(3)
w, f, r = [], [], []
for i in range(12):
    L.call("gc_bh_walk", tree.handle, 0.7)
    L.call("gc_bh_forces_async", tree.handle, 1.0, 1e-4)
    L.call("gc_bh_timings", tree.handle, L.ptr(tm, L.f64p))
    if i >= 2:
        w.append(tm[0])
        f.append(tm[1])
        r.append(tm[2])
inter = nbody.interactions(tree)
fm = statistics.median(f)
st = np.zeros(2, np.int64)
L.call("gc_bh_pair_stats", tree.handle, L.ptr(st, L.i64p))
print(f"{L.LIB_PATH.split('/')[-1]} {'staged' if staged else 'fused'}: walk {statistics.median(w):.3f} ms  reorg {statistics.median(r):.3f} ms  force {fm:.3f} ms  "
      f"{20 * inter / fm / 1e9:.2f} TFLOP/s ({inter} interactions) issued {st[0]} eff {inter / st[0]:.3f}")

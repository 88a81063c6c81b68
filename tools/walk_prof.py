"""Walk instrumentation (libgcharm built with -DWALK_PROF=1): active-bucket density per node visit."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2008_05712_b200 import _lib as L  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402
from paper_2008_05712_b200 import nbody  # noqa: E402

ps = gen.fp32_exact(gen.gen_particles(1_000_000, 42, clustering=0.6, dim=3))
tree = nbody.build_bucket_tree(ps, 8)
for _ in range(2):  # forces make the scheduling hints (heaviest walk groups first) used below
    L.call("gc_bh_walk", tree.handle, 0.7)
    L.call("gc_bh_forces_async", tree.handle, 1.0, 1e-4)
v = np.zeros(6, np.int64)
L.context().sync()
L.call("gc_debug_walk_prof", L.ptr(v, L.i64p), 1)
L.call("gc_bh_walk", tree.handle, 0.7)
L.context().sync()
L.call("gc_debug_walk_prof", L.ptr(v, L.i64p), 1)
print(f"node visits {v[0]}  mean active {v[1] / v[0]:.2f} of 64  one half empty {v[2] / v[0]:.3f}  "
      f"mean emitted {v[3] / v[0]:.2f}  first warp idle at {v[4] / 1e3:.1f} us, last warp done at {v[5] / 1e3:.1f} us")

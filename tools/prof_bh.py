"""Minimal BH driver for ncu captures: 1M clustered, theta 0.7; walk + forces x3
(fused force path), then walk + forces once in the staged mode (expand_kernel +
force_group_kernel) so one capture covers both."""
import sys

sys.path.insert(0, ".")
from paper_2008_05712_b200 import _lib as L  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402
from paper_2008_05712_b200 import nbody  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
tree = nbody.build_bucket_tree(ps, 8)
ctx = L.context()
for _ in range(3):
    L.call("gc_bh_walk", tree.handle, 0.7)
    L.call("gc_bh_forces_async", tree.handle, 1.0, 1e-4)
L.call("gc_bh_set_force_mode", tree.handle, 0)
L.call("gc_bh_walk", tree.handle, 0.7)
L.call("gc_bh_forces_async", tree.handle, 1.0, 1e-4)
ctx.sync()
print("interactions", nbody.interactions(tree))

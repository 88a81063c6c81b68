"""BH driver for ncu at configs[3] size on one GPU: Plummer 2^24, theta 0.7 (walk + fused force, twice)."""
import sys

sys.path.insert(0, ".")
from paper_2008_05712_b200 import _lib as L  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402
from paper_2008_05712_b200 import nbody  # noqa: E402

ps = gen.fp32_exact(gen.gen_plummer(1 << 24, 42))
tree = nbody.build_bucket_tree(ps, 8)
ctx = L.context()
for _ in range(2):
    L.call("gc_bh_walk", tree.handle, 0.7)
    L.call("gc_bh_forces_async", tree.handle, 1.0, 1e-4)
ctx.sync()
print("interactions", nbody.interactions(tree))

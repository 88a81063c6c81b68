"""Step time (walk + forces) per walk/force overlap mode (0 back to back, 1 PDL, 2 one persistent kernel), 1M clustered; forces must be identical."""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2008_05712_b200 import _lib as L  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402
from paper_2008_05712_b200 import nbody  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
tree = nbody.build_bucket_tree(ps, 8)
ctx = L.context()
ext = torch.cuda.ExternalStream(ctx.stream)
res = {}
for ov in (0, 1, 2, 0, 1, 2):
    L.call("gc_bh_set_overlap", tree.handle, ov)
    for _ in range(3):
        L.call("gc_bh_walk_forces_async", tree.handle, 0.7, 1.0, 1e-4)
    ctx.sync()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        L.call("gc_bh_walk_forces_async", tree.handle, 0.7, 1.0, 1e-4)
        e1.record(ext)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    f = np.zeros((len(ps.positions), 3))
    L.call("gc_bh_forces", tree.handle, 1.0, 1e-4, L.ptr(f, L.f64p))  # forces of the last step's lists (non-overlapped launch)
    L.call("gc_bh_walk_forces_async", tree.handle, 0.7, 1.0, 1e-4)
    ctx.sync()
    out = np.zeros((len(ps.positions), 3))
    L.call("gc_bh_get_forces", tree.handle, L.ptr(out, L.f64p))
    res.setdefault(ov, []).append(out)
    print(f"overlap={ov}: step {statistics.median(ts):.3f} ms (min {min(ts):.3f})", flush=True)
for ov in (1, 2):
    assert np.array_equal(res[0][0], res[ov][0]) and np.array_equal(res[0][1], res[ov][1]), f"forces differ (mode {ov})"
print("forces identical")

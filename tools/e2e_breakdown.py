"""Host-side breakdown of the BH end-to-end step (gc_bh_step pieces), wall clock."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2008_05712_b200 import _lib as L  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402
from paper_2008_05712_b200 import nbody  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
pos = torch.from_numpy(np.ascontiguousarray(ps.positions)).pin_memory().numpy()
m = torch.from_numpy(np.ascontiguousarray(ps.masses)).pin_memory().numpy()
out = torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy()
st = nbody.BHStep(8, 0.7, 1.0, 1e-4)
h = st.handle
for it in range(6):
    t0 = time.perf_counter()
    L.call("gc_bh_set_particles", h, n, 3, L.ptr(pos, L.f64p), L.ptr(m, L.f64p), 1.0, 8)
    t1 = time.perf_counter()
    L.call("gc_bh_walk", h, 0.7)
    t2 = time.perf_counter()
    L.call("gc_bh_forces", h, 1.0, 1e-4, L.ptr(out, L.f64p))
    t3 = time.perf_counter()
    st(pos, m, 1.0, out)
    t4 = time.perf_counter()
    print(f"iter {it}: set_particles {1e3*(t1-t0):.2f} ms  walk {1e3*(t2-t1):.2f} ms  forces+d2h {1e3*(t3-t2):.2f} ms"
          f"  | gc_bh_step {1e3*(t4-t3):.2f} ms", flush=True)

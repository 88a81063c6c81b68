"""configs[4]'s system on ONE B200: LJ FCC 126^3 x 4 = 8,001,504 atoms, 84^3 cells."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2008_05712_b200 import md  # noqa: E402
from paper_2008_05712_b200.generators import gen_lj_fcc  # noqa: E402

t0 = time.time()
s = gen_lj_fcc(126)
print("atoms", s.positions.shape[0], "cells", s.cells_xyz, f"gen {time.time() - t0:.1f} s", flush=True)
sysd = md.LJSystem(s)
f, e = sysd.forces()
print("force-only ms", sysd.dev.elapsed_ms(), "finite", bool(np.isfinite(f).all()), "E/atom", e.mean())
sysd.run(10)
for _ in range(2):
    print("10 steps ms", sysd.run(10))
p, v, c = sysd.state()
print("finite", bool(np.isfinite(p).all() and np.isfinite(v).all()), "KE/atom", 0.5 * (v ** 2).sum(1).mean())

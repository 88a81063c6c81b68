import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2008_05712_b200.generators import gen_lj_fcc
from paper_2008_05712_b200 import md, md_dist
from paper_2008_05712_b200 import _lib as L
inp = gen_lj_fcc(10, repeat_x=4)
s = md_dist.LJSlab(inp, 0, 24)
p0, v0, g0 = s.owned()
print("owned", len(g0), np.abs(p0 - inp.positions[g0]).max(), np.abs(v0 - inp.velocities[g0]).max())
hl, hr = s.halo_out()
print("halo", hl.shape, hr.shape)
s.set_halo(hr, hl)
s.advance(inp.dt)
torch.cuda.synchronize()
p1, v1, g1 = s.owned()
print("after advance: dv", np.abs(v1 - v0).max(), "dp", np.abs(p1 - p0).max())
w = md.LJSystem(inp); f, e = w.forces()
print("whole force max", np.abs(f).max())

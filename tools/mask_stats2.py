"""Sub-group lane mappings of the 32-target force groups (CPU design study):
lanes = T consecutive targets x 32/T record phases; each sub-group evaluates
the records of the union entries some of its targets' buckets use."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as orc  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
nb = len(t.buckets)
b0 = nb // 3 - (nb // 3) % 64
b1 = b0 + 12800
ol = orc.build_interaction_lists(t, 0.7, bucket_range=(b0, b1))
pc = t.pcount
nbk = pc[t.buckets]
useful = sum(int(nbk[b]) * int(ol.item_count[b]) for b in range(b0, b1))


def groups(wb0, wb1, T=32):
    out, cur, tg = [], [], 0
    for b in range(wb0, wb1):
        c = int(nbk[b])
        if cur and tg + c > T:
            out.append(cur)
            cur, tg = [], 0
        cur.append(b)
        tg += c
    if cur:
        out.append(cur)
    return out


res = {T: [0, 0] for T in (32, 16, 8, 4)}
for wb in range(b0, b1, 64):
    for g in groups(wb, min(b1, wb + 64)):
        tb = np.concatenate([[j] * int(nbk[b]) for j, b in enumerate(g)])  # bucket of each target lane
        ent = {}
        for j, b in enumerate(g):
            w = ol.walk_order(b)
            k = ol.kind[ol.ptr[b]:ol.ptr[b + 1]]
            for x, kk in zip(w.tolist(), k.tolist()):
                e = ent.setdefault(x, [0, 0])
                e[kk] |= 1 << j
        for T in res:
            ph = 32 // T
            for s in range(0, len(tb), T):
                sub = 0
                for j in tb[s:s + T]:
                    sub |= 1 << int(j)
                R = sum((1 if a & sub else 0) + (int(pc[x]) if p & sub else 0) for x, (a, p) in ent.items())
                res[T][0] += R
                res[T][1] += 32 * -(-R // ph)
for T, (R, iss) in res.items():
    print(f"T={T:2d} x {32 // T} phases: eff {useful / iss:.3f} records/useful {R / useful:.4f}")

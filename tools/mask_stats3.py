"""Concurrent sub-stream design study (CPU): the warp's 32 target lanes are cut
into S slices of 32/S lanes; slice s evaluates only the union records whose
bucket mask meets its lanes' buckets, all slices stepping together (a slice
that runs dry idles), so a force group costs 32 x max_s R_s lane-pairs.
Reports useful / issued for S = 1, 2, 4, 8 and the record copies per union
record.  Usage: python tools/mask_stats3.py [n]"""
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


SS = (1, 2, 4, 8)
iss = {s: 0 for s in SS}
cop = {s: 0 for s in SS}
union = 0
for wb in range(b0, b1, 64):
    for g in groups(wb, min(b1, wb + 64)):
        tb = np.concatenate([[j] * int(nbk[b]) for j, b in enumerate(g)])
        ent = {}
        for j, b in enumerate(g):
            w = ol.walk_order(b)
            k = ol.kind[ol.ptr[b]:ol.ptr[b + 1]]
            for x, kk in zip(w.tolist(), k.tolist()):
                e = ent.setdefault(x, [0, 0])
                e[kk] |= 1 << j
        union += sum((1 if a else 0) + (int(pc[x]) if p else 0) for x, (a, p) in ent.items())
        for S in SS:
            L = 32 // S
            rs = []
            for s in range(S):
                sub = 0
                for j in tb[s * L:(s + 1) * L]:
                    sub |= 1 << int(j)
                rs.append(sum((1 if a & sub else 0) + (int(pc[x]) if p & sub else 0) for x, (a, p) in ent.items())
                          if sub else 0)
            iss[S] += 32 * max(rs)
            cop[S] += sum(rs)
for S in SS:
    print(f"S={S} slices of {32 // S} lanes: eff {useful / iss[S]:.3f}  copies/union record {cop[S] / union:.2f}")

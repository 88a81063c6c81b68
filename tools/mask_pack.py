"""Slot packing study: records whose bucket sets are disjoint share one
consumer step (each lane picks the record of its bucket).  Schemes:
  S0: one record per step (current);
  S1: single-bucket records packed (k-th single record of every bucket share a step), others alone;
  S2: greedy first-fit packing of all records by bucket set (window of W records)."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from oracle import oracle as orc
from paper_2008_05712_b200 import generators as gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
nb = len(t.buckets)
b0 = nb // 3 - (nb // 3) % 64
b1 = b0 + 6400
ol = orc.build_interaction_lists(t, 0.7, bucket_range=(b0, b1))
pc = t.pcount
nbk = pc[t.buckets]
def groups(wb0, wb1, T=32):
    out, cur, tg = [], [], 0
    for b in range(wb0, wb1):
        c = int(nbk[b])
        if cur and tg + c > T:
            out.append(cur); cur, tg = [], 0
        cur.append(b); tg += c
    if cur: out.append(cur)
    return out
useful = 0; s0 = s1 = 0; s2 = {32: 0, 128: 0}; nsingle = nrec = 0
for wb in range(b0, b1, 64):
    for g in groups(wb, min(b1, wb + 64)):
        ent = {}
        for j, b in enumerate(g):
            w = ol.walk_order(b); k = ol.kind[ol.ptr[b]:ol.ptr[b + 1]]
            for x, kk in zip(w.tolist(), k.tolist()):
                e = ent.setdefault(x, [0, 0]); e[kk] |= 1 << j
        recs = []  # bucket mask per record (in stream order)
        for x, (a, p) in ent.items():
            if a: recs.append(a)
            if p: recs += [p] * int(pc[x])
        tgt = [int(nbk[b]) for b in g]
        useful += sum(sum(tgt[j] for j in range(len(g)) if m >> j & 1) for m in recs)
        nrec += len(recs)
        s0 += len(recs)
        single = [m for m in recs if m & (m - 1) == 0]
        multi = len(recs) - len(single)
        nsingle += len(single)
        per_b = np.bincount([m.bit_length() - 1 for m in single], minlength=len(g)) if single else np.zeros(1)
        s1 += multi + int(per_b.max())
        for W in s2:
            for w0 in range(0, len(recs), W):
                slots = []
                for m in recs[w0:w0 + W]:
                    for i, sm in enumerate(slots):
                        if sm & m == 0:
                            slots[i] |= m; break
                    else:
                        slots.append(m)
                s2[W] += len(slots)
print(f"records {nrec}, single-bucket {nsingle / nrec:.3f}")
print(f"S0 eff {useful / (32 * s0):.3f}  S1 eff {useful / (32 * s1):.3f} (steps x{s1 / s0:.3f})")
for W in s2: print(f"S2 W={W} eff {useful / (32 * s2[W]):.3f} (steps x{s2[W] / s0:.3f})")

"""Force-group mask statistics from oracle lists (CPU; design study for the
force kernel): for several target-group sizes T (lanes = T targets x 32/T
record phases), the issued lane-pairs vs useful interactions and the records
gathered.  Usage: python tools/mask_stats.py [n] [b0 b1]"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as orc  # noqa: E402
from paper_2008_05712_b200 import generators as gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ps = gen.fp32_exact(gen.gen_particles(n, 42, clustering=0.6, dim=3))
t0 = time.time()
t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
nb = len(t.buckets)
b0, b1 = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (nb // 3, nb // 3 + 12800)
b0 -= b0 % 64
ol = orc.build_interaction_lists(t, 0.7, bucket_range=(b0, b1))
print(f"tree+lists {time.time() - t0:.1f}s, buckets {nb}, sample [{b0},{b1})")
pc = t.pcount
nbk = pc[t.buckets]


def groups(wb0, wb1, T):
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


useful = 0
for b in range(b0, b1):
    useful += int(nbk[b]) * int(ol.item_count[b])
for T in (32, 16, 8):
    ph = 32 // T
    issued = rec = issued_pad = 0
    for wb in range(b0, b1, 64):
        for g in groups(wb, min(b1, wb + 64), T):
            acc, opn = set(), set()
            for b in g:
                w = ol.walk_order(b)
                k = ol.kind[ol.ptr[b]:ol.ptr[b + 1]]
                acc.update(w[k == 0].tolist())
                opn.update(w[k == 1].tolist())
            R = len(acc) + int(sum(pc[x] for x in opn))
            rec += R
            issued += 32 * -(-R // ph)
            issued_pad += 32 * -(-(-(-R // 16) * 16) // ph)
    print(f"T={T:2d} x {ph} phases: records {rec:,} issued {issued:,} eff {useful / issued:.3f} "
          f"(padded16 {useful / issued_pad:.3f}) records/useful {rec / useful:.4f}")
print(f"useful {useful:,}")

# split design: records every bucket of the group uses are broadcast (all
# lanes useful); the rest go through per-bucket index lists, lane = target,
# iterations = max over the group's buckets of its partial-list length
for T in (32,):
    full_rec = part_iters = part_useful = full_useful = ntg = 0
    ic_iters = 0
    for wb in range(b0, b1, 64):
        for g in groups(wb, min(b1, wb + 64), T):
            cnt = {}
            for b in g:
                w = ol.walk_order(b)
                k = ol.kind[ol.ptr[b]:ol.ptr[b + 1]]
                for x, kk in zip(w.tolist(), k.tolist()):
                    cnt[(x, kk)] = cnt.get((x, kk), 0) + 1
            nbg = len(g)
            full = {e for e, c in cnt.items() if c == nbg}
            fr = sum(1 if kk == 0 else int(pc[x]) for x, kk in full)
            tg = int(sum(nbk[b] for b in g))
            ntg += tg
            full_rec += fr
            full_useful += fr * tg
            lens = []
            for b in g:
                w = ol.walk_order(b)
                k = ol.kind[ol.ptr[b]:ol.ptr[b + 1]]
                L = sum(1 if kk == 0 else int(pc[x]) for x, kk in zip(w.tolist(), k.tolist()) if (x, kk) not in full)
                lens.append(L)
                part_useful += L * int(nbk[b])
            part_iters += max(lens)
            ic_iters += max(int(ol.item_count[b]) for b in g)
    print(f"split T=32: full-mask useful {full_useful / useful:.3f} of useful; full issue eff "
          f"{full_useful / (32 * full_rec):.3f}; partial per-lane eff {part_useful / (32 * part_iters):.3f}; "
          f"overall {useful / (32 * (full_rec + part_iters)):.3f}; all-per-lane eff {useful / (32 * ic_iters):.3f}")

# per-lane design on a window of W consecutive union records: iterations per
# window = max over the group's buckets of the records it uses in the window
for W in (32, 64, 128, 256, 1 << 30):
    iters = 0
    for wb in range(b0, b1, 64):
        for g in groups(wb, min(b1, wb + 64), 32):
            ents = {}
            order = []
            for j, b in enumerate(g):
                w = ol.walk_order(b)
                k = ol.kind[ol.ptr[b]:ol.ptr[b + 1]]
                for x, kk in zip(w.tolist(), k.tolist()):
                    if x not in ents:
                        ents[x] = [0, 0]
                        order.append(x)
                    ents[x][kk] |= 1 << j
            # records in a plausible union order (preorder of node ids is close to emission order)
            masks = []
            for x in sorted(order):
                a, p = ents[x]
                if a:
                    masks.append(a)
                if p:
                    masks.extend([p] * int(pc[x]))
            m = np.array(masks, np.int64)
            for s in range(0, len(m), min(W, len(m) if len(m) else 1)):
                mw = m[s:s + W]
                iters += max(int(((mw >> j) & 1).sum()) for j in range(len(g)))
    print(f"per-lane window {W}: eff {useful / (32 * iters):.3f}")

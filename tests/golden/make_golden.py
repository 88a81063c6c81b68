"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the dev container only (the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports hetero-rt from /root/reference/pkg/src, runs the reference's own
functions on small seeded inputs (float32-exact, as the B200 path consumes)
and writes their outputs.  Large cases are stored as sha256 digests of the
exact arrays ("checksum of checksums").  Fixtures pin the oracle/ restatement
(tests/test_oracle_golden.py) and, on the GPU, the product (tests/test_*_gpu.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from hetero_rt import kernels as rk  # noqa: E402
from hetero_rt.aggregator import AggregatorState, observe_arrival, poll_combine  # noqa: E402
from hetero_rt.memory import DeviceMemory, MemoryMode  # noqa: E402
from hetero_rt.runtime import WorkRequest  # noqa: E402
from hetero_rt.scheduler import PerfEstimate, partition_queue  # noqa: E402
from hetero_rt.workloads import md as rmd  # noqa: E402
from hetero_rt.workloads import nbody as rnb  # noqa: E402

from paper_2008_05712_b200 import generators as gen  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def ref_ps(ps):
    return rnb.ParticleSet(positions=ps.positions.copy(), masses=ps.masses.copy(),
                           velocities=ps.velocities.copy(), box=ps.box)


def tree_arrays(tree, dim):
    nn = len(tree.nodes)
    center = np.array([n.center for n in tree.nodes], dtype=np.float64).reshape(nn, dim)
    half = np.array([n.half_size for n in tree.nodes])
    mass = np.array([n.mass for n in tree.nodes])
    com = np.array([n.com for n in tree.nodes], dtype=np.float64).reshape(nn, dim)
    first_child = np.array([n.children[0].node_id if n.children else -1 for n in tree.nodes], np.int64)
    n_child = np.array([len(n.children) for n in tree.nodes], np.int32)
    pcount = np.array([len(n.particle_idx) for n in tree.nodes], np.int64)
    buckets = np.array([b.node_id for b in tree.buckets], np.int64)
    pidx = np.concatenate([b.particle_idx for b in tree.buckets]).astype(np.int64)
    return dict(center=center, half=half, mass=mass, com=com, first_child=first_child, n_child=n_child,
                pcount=pcount, buckets=buckets, pidx=pidx)


def list_arrays(lists):
    ptr = np.zeros(len(lists) + 1, np.int64)
    ids, kind, ic = [], [], []
    for i, il in enumerate(lists):
        nodes = set(il.node_interactions)
        ids.extend(il.walk_order)
        kind.extend(0 if b in nodes else 1 for b in il.walk_order)
        ptr[i + 1] = ptr[i] + len(il.walk_order)
        ic.append(il.item_count)
        # node/particle subsequences must be the walk order filtered by kind
        assert [b for b in il.walk_order if b in nodes] == list(il.node_interactions)
    return dict(ptr=ptr, ids=np.array(ids, np.int64), kind=np.array(kind, np.int8),
                item_count=np.array(ic, np.int64))


def nbody_case(name, ps, bucket, thetas, forces_theta, store_full=True):
    t0 = time.time()
    rps = ref_ps(ps)
    dim = ps.positions.shape[1]
    tree = rnb.build_bucket_tree(rps, bucket)
    out = dict(positions=ps.positions, masses=ps.masses, bucket_size=np.int64(bucket), box=np.float64(ps.box))
    out.update({f"tree_{k}": v for k, v in tree_arrays(tree, dim).items()})
    digests = {"tree": sha(*[out[f"tree_{k}"] for k in ("center", "half", "mass", "com", "first_child",
                                                         "n_child", "pcount", "buckets", "pidx")])}
    for th in thetas:
        lists = rnb.build_interaction_lists(tree, th, rps)
        la = list_arrays(lists)
        tag = f"theta{th:g}".replace(".", "p")
        digests[f"lists_{tag}"] = sha(la["ptr"], la["ids"], la["kind"], la["item_count"])
        out.update({f"lists_{tag}_{k}": v for k, v in la.items()})
        if th == forces_theta:
            f = rnb.eval_forces(tree, lists, rps)
            out[f"forces_{tag}"] = f
            digests[f"forces_{tag}"] = sha(f)
    if store_full:
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {len(tree.nodes)} nodes, {len(tree.buckets)} buckets, {time.time() - t0:.1f}s")
    return digests


def main():
    meta = {"reference": "hetero-rt @ /root/reference/pkg/src", "numpy": np.__version__,
            "numba": rk.NUMBA_ENABLED}
    digests = {}

    # generator identity with the reference
    for (n, seed, cl, dim) in [(300, 9, 0.5, 2), (2048, 12, 0.6, 3), (1000, 3, 0.0, 3)]:
        a = gen.gen_particles(n, seed, cl, dim)
        b = rnb.gen_particles(n, seed, cl, dim)
        assert np.array_equal(a.positions, b.positions) and np.array_equal(a.masses, b.masses)
    g_md = gen.gen_md_system((10, 10), 24, 1.0, 7)
    r_md, _ = rmd.gen_md_system((10, 10), 24, 1.0, 7)
    assert np.array_equal(g_md[0], r_md.positions) and np.array_equal(g_md[2], r_md.patch_of)

    # --- N-body trees / lists / forces (small: full arrays) ---------------------
    ps = gen.fp32_exact(gen.gen_particles(300, 9, 0.5, 2))
    digests["nbody2d_300"] = nbody_case("nbody2d_300", ps, 8, [0.0, 0.3, 0.7], 0.7)
    ps = gen.fp32_exact(gen.gen_particles(2048, 12, 0.6, 3))
    digests["nbody3d_2048"] = nbody_case("nbody3d_2048", ps, 8, [0.0, 0.7], 0.7)
    ps = gen.fp32_exact(gen.gen_plummer(4096, 42))
    digests["plummer3d_4096"] = nbody_case("plummer3d_4096", ps, 8, [0.7], 0.7)
    # --- config 1 (Plummer 16K, theta 0.7): digests only -------------------------
    ps = gen.fp32_exact(gen.gen_plummer(16384, 42))
    digests["plummer3d_16384"] = nbody_case("plummer3d_16384", ps, 8, [0.7], 0.7, store_full=False)

    # --- kernels: coincident sources, MD pair kernels ----------------------------
    rng = np.random.default_rng(99)
    ppos = rng.uniform(0, 1, size=(10, 3)).astype(np.float32).astype(np.float64)
    pmass = rng.uniform(0.5, 1.5, size=10).astype(np.float32).astype(np.float64)
    spos = np.vstack([rng.uniform(0, 1, size=(40, 3)).astype(np.float32).astype(np.float64), ppos[:3]])
    smass = rng.uniform(0.5, 1.5, size=43).astype(np.float32).astype(np.float64)
    ffp = rk.forces_from_points(ppos, pmass, spos, smass, 1.0, 1e-4)
    ffp0 = rk.forces_from_points(ppos, pmass, spos, smass, 1.0, 0.0)
    a = rng.uniform(0, 2, size=(15, 2))
    b = rng.uniform(0, 2, size=(12, 2))
    fa, fb = rk.md_cross_forces(a, b, 1.0, 25.0)
    sp = rng.uniform(0, 1.5, size=(30, 2))
    fs = rk.md_self_forces(sp, 1.0, 25.0)
    dpos = rng.uniform(0, 1, size=(256, 3)).astype(np.float32).astype(np.float64)
    dmass = rng.uniform(0.5, 1.5, size=256).astype(np.float32).astype(np.float64)
    dfor = rk.direct_forces(dpos, dmass, 1.0, 1e-4)
    runs_in = [rng.integers(0, 300, size=int(rng.integers(1, 200))).astype(np.int64) for _ in range(50)]
    runs_out = np.array([rk.count_address_runs(x, 16) for x in runs_in], np.int64)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), ppos=ppos, pmass=pmass, spos=spos, smass=smass,
                        ffp=ffp, ffp_eps0=ffp0, md_a=a, md_b=b, md_fa=fa, md_fb=fb, md_self_pos=sp,
                        md_self_f=fs, direct_pos=dpos, direct_mass=dmass, direct_f=dfor,
                        runs_lens=np.array([len(x) for x in runs_in]), runs_in=np.concatenate(runs_in),
                        runs_out=runs_out)

    # --- 2-D soft MD (compute_forces + md_step) -----------------------------------
    md_out = {}
    for periodic in (False, True):
        grid, _ = rmd.gen_md_system((10, 10), 24, 1.0, 7)
        tag = "per" if periodic else "wall"
        md_out[f"{tag}_pos0"] = grid.positions.copy()
        md_out[f"{tag}_vel0"] = grid.velocities.copy()
        md_out[f"{tag}_patch0"] = grid.patch_of.copy()
        md_out[f"{tag}_f0"] = rmd.compute_forces(grid, 25.0, periodic)
        for s in range(3):
            rmd.md_step(grid, 0.08, 25.0, periodic)
        md_out[f"{tag}_pos3"] = grid.positions.copy()
        md_out[f"{tag}_vel3"] = grid.velocities.copy()
        md_out[f"{tag}_patch3"] = grid.patch_of.copy()
        md_out[f"{tag}_f3"] = rmd.compute_forces(grid, 25.0, periodic)
    np.savez_compressed(os.path.join(HERE, "md2d.npz"), **md_out)
    grid, _ = rmd.gen_md_system((67, 67), 24, 1.0, 7)
    digests["md2d_67x67"] = {"forces": sha(rmd.compute_forces(grid, 25.0, False)), "n": int(len(grid.positions))}

    # --- data manager plans ------------------------------------------------------
    dm_cases = []
    def run_dm(mode, cap, slot, batches, release_after=True):
        mem = DeviceMemory(cap, slot, MemoryMode(mode))
        rec = []
        for i, (members, now) in enumerate(batches):
            try:
                plan, layout = mem.build_plan([list(m) for m in members], now)
                rec.append(dict(ok=True, to_transfer=[b for b, _ in plan.to_transfer],
                                total_bytes=plan.total_bytes, indirection_bytes=plan.indirection_bytes,
                                addresses=layout.addresses.tolist(), bounds=layout.member_bounds.tolist(),
                                indirect=layout.indirect, transactions=layout.member_transactions(),
                                table=sorted((b, mem.table.get(b).slot_index) for b in mem.table.buffers())))
                if release_after:
                    mem.release_batch([list(m) for m in members])
            except Exception as e:  # CapacityError
                rec.append(dict(ok=False, error=type(e).__name__))
        return rec

    fig1 = [([[2, 5, 7]], 0.0), ([[2, 3, 5, 7, 8]], 1.0)]
    for mode in ("redundant", "reuse", "reuse_sorted"):
        dm_cases.append(dict(name=f"fig1_{mode}", mode=mode, cap=1 << 16, slot=256, batches=fig1,
                             release=True, result=run_dm(mode, 1 << 16, 256, fig1)))
    fig1s = [([[2, 5, 7]], 0.0), ([[7, 3, 2, 8, 5]], 1.0)]
    dm_cases.append(dict(name="fig1_sorted_perm", mode="reuse_sorted", cap=1 << 16, slot=256, batches=fig1s,
                         release=True, result=run_dm("reuse_sorted", 1 << 16, 256, fig1s)))
    rng = np.random.default_rng(31)
    for case in range(12):
        batches = []
        universe = int(rng.integers(50, 400))
        for step in range(int(rng.integers(5, 25))):
            members = []
            for _ in range(int(rng.integers(1, 6))):
                idx = []
                for _ in range(int(rng.integers(1, 5))):
                    s0 = int(rng.integers(0, universe - 12))
                    idx.extend(range(s0, s0 + int(rng.integers(2, 12))))
                idx = list(dict.fromkeys(idx))
                rng.shuffle(idx)
                members.append([int(x) for x in idx])
            batches.append((members, float(step) + float(rng.uniform(0, 0.5))))
        cap_slots = int(rng.choice([32, 64, 128, 4096]))
        for mode in ("redundant", "reuse", "reuse_sorted"):
            dm_cases.append(dict(name=f"rand{case}_{mode}", mode=mode, cap=cap_slots * 64, slot=64,
                                 batches=batches, release=True,
                                 result=run_dm(mode, cap_slots * 64, 64, batches)))
    # pinned (never released) batches to force CapacityError paths
    batches = [([[1, 2]], 0.0), ([[3]], 1.0), ([[4, 5]], 2.0)]
    dm_cases.append(dict(name="pinned_reuse", mode="reuse", cap=2 * 64, slot=64, batches=batches,
                         release=False, result=run_dm("reuse", 2 * 64, 64, batches, release_after=False)))
    with open(os.path.join(HERE, "dm_plans.json"), "w") as fh:
        json.dump(dm_cases, fh)

    # --- combining trigger emissions + partitioner ------------------------------
    rng = np.random.default_rng(303)
    agg = []
    for _ in range(60):
        n = int(rng.integers(20, 160))
        t = 0.0
        arrivals = []
        for i in range(n):
            t += float(rng.uniform(3.0, 20.0)) if rng.random() < 0.08 else float(rng.uniform(0.0, 0.6))
            arrivals.append((t, i))
        max_size = int(rng.integers(2, 24))
        polls = [float(x) for x in np.arange(0.0, arrivals[-1][0] + 60.0, 1.0)]
        state = AggregatorState("force", max_size=max_size)
        got, ai = [], 0
        for pt in sorted(set(polls) | {a for a, _ in arrivals}):
            while ai < len(arrivals) and arrivals[ai][0] <= pt:
                at, aid = arrivals[ai]
                state.pending.append(WorkRequest(aid, 0, "force", [aid], 1, at))
                observe_arrival(state, at)
                ai += 1
            while True:
                bt = poll_combine(state, pt)
                if bt is None:
                    break
                got.append([pt, [m.id for m in bt.members]])
        agg.append(dict(arrivals=arrivals, max_size=max_size, polls=polls, emissions=got))
    parts = []
    for _ in range(100):
        items = [int(x) for x in rng.integers(1, 50, size=int(rng.integers(1, 30)))]
        share = float(rng.uniform(0, 1))
        near = bool(rng.random() < 0.5)
        q = [WorkRequest(i, 0, "force", [0], w, 0.0) for i, w in enumerate(items)]
        p = partition_queue(q, PerfEstimate(), cpu_share=share, nearest_target=near)
        parts.append(dict(items=items, share=share, nearest=near, cut=len(p.cpu_set)))
    with open(os.path.join(HERE, "aggregator.json"), "w") as fh:
        json.dump(dict(emissions=agg, partitions=parts), fh)

    meta["digests"] = digests
    with open(os.path.join(HERE, "digests.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("done")


if __name__ == "__main__":
    main()

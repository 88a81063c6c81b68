"""GPU parity of the Barnes-Hut path (device tree/walk/forces) against the
reference's golden fixtures and the CPU oracle.

Bars: tree arrays, interaction lists (walk_order, kinds, item_count) are
bit-exact; forces match float64 within FORCE_RTOL, measured per particle as
||F_gpu - F_ref||_2 / ||F_ref||_2 (max over all particles).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

FORCE_RTOL = 1e-5


def rel_err(a, b):
    return np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def nb():
    from paper_2008_05712_b200 import nbody
    return nbody


def tag(th):
    return f"theta{th:g}".replace(".", "p")


CASES = [("nbody2d_300", [0.0, 0.3, 0.7], 0.7), ("nbody3d_2048", [0.0, 0.7], 0.7),
         ("plummer3d_4096", [0.7], 0.7)]


@pytest.mark.parametrize("name,thetas,ftheta", CASES)
def test_golden_tree_lists_forces(nb, name, thetas, ftheta):
    from paper_2008_05712_b200.generators import ParticleSet
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    ps = ParticleSet(g["positions"], g["masses"], np.zeros_like(g["positions"]), float(g["box"]))
    tree = nb.build_bucket_tree(ps, int(g["bucket_size"]))
    for k in ("center", "half", "mass", "com", "first_child", "n_child"):
        np.testing.assert_array_equal(getattr(tree, k), g[f"tree_{k}"], err_msg=k)
    np.testing.assert_array_equal(tree.bucket_ids, g["tree_buckets"])
    np.testing.assert_array_equal(tree.pidx, g["tree_pidx"])
    for th in thetas:
        lists = nb.build_interaction_lists(tree, th, ps)
        ptr, ids, kind, ic = lists.csr()
        np.testing.assert_array_equal(ptr, g[f"lists_{tag(th)}_ptr"])
        np.testing.assert_array_equal(ids, g[f"lists_{tag(th)}_ids"])
        np.testing.assert_array_equal(kind, g[f"lists_{tag(th)}_kind"])
        np.testing.assert_array_equal(ic, g[f"lists_{tag(th)}_item_count"])
        if th == ftheta:
            f = nb.eval_forces(tree, lists, ps)
            assert rel_err(f, g[f"forces_{tag(th)}"]).max() <= FORCE_RTOL


def test_reference_objects_via_member_kernel(nb):
    """Lists handed in from the host runtime (reference-style objects) run on
    the per-work-request kernel and give the same forces."""
    from paper_2008_05712_b200.generators import ParticleSet
    g = np.load(os.path.join(GOLDEN, "nbody3d_2048.npz"))
    ps = ParticleSet(g["positions"], g["masses"], np.zeros_like(g["positions"]), 1.0)
    tree = nb.build_bucket_tree(ps, 8)
    csr = (g["lists_theta0p7_ptr"], g["lists_theta0p7_ids"], g["lists_theta0p7_kind"])
    f = nb.eval_forces(tree, csr, ps)
    assert rel_err(f, g["forces_theta0p7"]).max() <= FORCE_RTOL
    dev = nb.build_interaction_lists(tree, 0.7, ps)
    objs = list(dev)  # reference-shaped InteractionList objects
    f2 = nb.eval_forces(tree, objs, ps)
    assert rel_err(f2, g["forces_theta0p7"]).max() <= FORCE_RTOL
    f3 = nb.eval_forces(tree, dev, ps)  # device lists again (re-walk after set_lists)
    assert rel_err(f3, g["forces_theta0p7"]).max() <= FORCE_RTOL


def test_plummer16k_config1_digests(nb):
    from paper_2008_05712_b200 import generators as gen
    from oracle import oracle as orc
    d = json.load(open(os.path.join(GOLDEN, "digests.json")))["digests"]["plummer3d_16384"]
    ps = gen.fp32_exact(gen.gen_plummer(16384, 42))
    tree = nb.build_bucket_tree(ps, 8)
    pc = np.where(tree.first_child < 0, tree.pcount, 0)
    assert sha(tree.center, tree.half, tree.mass, tree.com, tree.first_child, tree.n_child, pc,
               tree.bucket_ids, tree.pidx) == d["tree"]
    lists = nb.build_interaction_lists(tree, 0.7, ps)
    ptr, ids, kind, ic = lists.csr()
    assert sha(ptr, ids, kind, ic) == d["lists_theta0p7"]
    f = nb.eval_forces(tree, lists, ps)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    ref = orc.eval_forces(ot, orc.build_interaction_lists(ot, 0.7), ps.positions, ps.masses)
    assert sha(ref) == d["forces_theta0p7"]  # oracle == reference bits
    assert rel_err(f, ref).max() <= FORCE_RTOL


def test_clustered_1m_config3_full_size(nb):
    """configs[2]: clustered 1M, theta 0.7 -- lists bit-exact against the
    oracle (itself pinned to the reference), forces within FORCE_RTOL."""
    from paper_2008_05712_b200 import generators as gen
    from oracle import oracle as orc
    ps = gen.fp32_exact(gen.gen_particles(1_000_000, 42, clustering=0.6, dim=3))
    tree = nb.build_bucket_tree(ps, 8)
    lists = nb.build_interaction_lists(tree, 0.7, ps)
    f = nb.eval_forces(tree, lists, ps)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    ol = orc.build_interaction_lists(ot, 0.7)
    ptr, ids, kind, ic = lists.csr()
    assert np.array_equal(ptr, ol.ptr)
    assert np.array_equal(ic, ol.item_count)
    assert np.array_equal(ids, ol.ids)
    assert np.array_equal(kind, ol.kind)
    ref = orc.eval_forces(ot, ol, ps.positions, ps.masses)
    e = rel_err(f, ref)
    print(f"1M clustered: median {np.median(e):.2e} p99.9 {np.percentile(e, 99.9):.2e} max {e.max():.2e}")
    assert e.max() <= FORCE_RTOL
    assert nb.interactions(tree) == int((tree.pcount[tree.bucket_ids] * ic).sum())


def test_theta_zero_equals_direct(nb):
    from paper_2008_05712_b200 import generators as gen
    ps = gen.fp32_exact(gen.gen_particles(512, 15, clustering=0.5, dim=3))
    tree = nb.build_bucket_tree(ps, 8)
    lists = nb.build_interaction_lists(tree, 0.0, ps)
    for il in lists:
        assert il.node_interactions == []
    f = nb.eval_forces(tree, lists, ps)
    exact = nb.direct_force_oracle(ps)
    assert rel_err(f, exact).max() <= FORCE_RTOL


def test_edge_cases(nb):
    from paper_2008_05712_b200.generators import ParticleSet
    # single particle, root is a bucket
    ps = ParticleSet(np.array([[0.25, 0.75]]), np.ones(1), np.zeros((1, 2)), 1.0)
    t = nb.build_bucket_tree(ps, 8)
    assert len(t.buckets) == 1 and t.root.is_bucket
    f = nb.eval_forces(t, nb.build_interaction_lists(t, 0.5, ps), ps)
    assert np.all(f == 0.0)
    # four quadrants, bucket size 1 (test_workloads.py:40-48)
    pts = np.array([[0.2, 0.2], [0.8, 0.2], [0.2, 0.8], [0.8, 0.8]])
    ps = ParticleSet(pts, np.ones(4), np.zeros((4, 2)), 1.0)
    t = nb.build_bucket_tree(ps, 1)
    assert len(t.buckets) == 4
    lists = nb.build_interaction_lists(t, 100.0, ps)
    assert all(len(il.walk_order) <= 4 for il in lists)
    # two-body Newton with eps = 0 (test_workloads.py:112-121)
    ps = ParticleSet(np.array([[0.0, 0.0], [1.0, 0.0]]), np.ones(2), np.zeros((2, 2)), 2.0)
    f = nb.direct_force_oracle(ps, g=1.0, eps=0.0)
    np.testing.assert_allclose(f, [[1.0, 0.0], [-1.0, 0.0]], atol=1e-12)
    t = nb.build_bucket_tree(ps, 1)
    f = nb.eval_forces(t, nb.build_interaction_lists(t, 0.0, ps), ps, g=1.0, eps=0.0)
    np.testing.assert_allclose(f, [[1.0, 0.0], [-1.0, 0.0]], rtol=1e-6)
    # coincident particles need softening
    ps = ParticleSet(np.array([[0.5, 0.5], [0.5, 0.5]]), np.ones(2), np.zeros((2, 2)), 1.0)
    with pytest.raises(Exception):
        nb.direct_force_oracle(ps, eps=0.0)
    with pytest.raises(ValueError):
        nb.build_bucket_tree(ps, 0)


def test_kernels_api_bit_exact():
    from paper_2008_05712_b200 import kernels as kn
    g = np.load(os.path.join(GOLDEN, "kernels.npz"))
    np.testing.assert_array_equal(kn.forces_from_points(g["ppos"], g["pmass"], g["spos"], g["smass"], 1.0, 1e-4),
                                  g["ffp"])
    np.testing.assert_array_equal(kn.forces_from_points(g["ppos"], g["pmass"], g["spos"], g["smass"], 1.0, 0.0),
                                  g["ffp_eps0"])
    fa, fb = kn.md_cross_forces(g["md_a"], g["md_b"], 1.0, 25.0)
    np.testing.assert_array_equal(fa, g["md_fa"])
    np.testing.assert_array_equal(fb, g["md_fb"])
    np.testing.assert_array_equal(kn.md_self_forces(g["md_self_pos"], 1.0, 25.0), g["md_self_f"])
    np.testing.assert_array_equal(kn.direct_forces(g["direct_pos"], g["direct_mass"], 1.0, 1e-4), g["direct_f"])
    off = np.concatenate([[0], np.cumsum(g["runs_lens"])])
    for i in range(len(g["runs_lens"])):
        assert kn.count_address_runs(g["runs_in"][off[i]:off[i + 1]], 16) == g["runs_out"][i]
    assert kn.count_address_runs(np.arange(40), 16) == 3
    assert kn.count_address_runs(np.arange(0, 32, 2), 16) == 16


@pytest.mark.parametrize("name,n,seed,cl,dim", [("clustered_1m", 1_000_000, 42, 0.6, 3), ("uniform2d", 20000, 3, 0.0, 2),
                                                ("plummer_200k", 200_000, 42, None, 3)])
def test_device_build_equals_oracle_tree(nb, name, n, seed, cl, dim):
    """The GPU tree build equals the float64 oracle's tree bit for bit at full
    size (node geometry, mass / COM bits, child ranges, bucket order and the
    particle order inside every bucket); the oracle is pinned to the reference
    by the golden tests above."""
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    ps = gen.fp32_exact(gen.gen_plummer(n, seed) if cl is None else gen.gen_particles(n, seed, cl, dim))
    a = nb.build_bucket_tree(ps, 8)
    o = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    for k in ("center", "half", "mass", "com", "first_child", "n_child", "pcount"):
        np.testing.assert_array_equal(np.asarray(getattr(a, k)).reshape(np.shape(getattr(o, k))), getattr(o, k),
                                      err_msg=k)
    np.testing.assert_array_equal(a.bucket_ids, o.buckets)
    for b in o.buckets[:: max(1, len(o.buckets) // 5000)]:
        np.testing.assert_array_equal(a.particle_idx(int(b)), o.particle_idx(int(b)))


def _edge_set(case):
    from paper_2008_05712_b200 import generators as gen
    rng = np.random.default_rng(7)
    box, dim = 1.0, 3
    if case in ("n1", "n8", "n9"):
        pos = rng.uniform(0.0, 1.0, size=(int(case[1:]), 3))
    elif case == "coincident":  # 20 identical points: a level-nlev bucket, the deep sort path
        pos = np.concatenate([rng.uniform(0.0, 1.0, size=(3000, 3)), np.full((20, 3), 0.3141592)])
    elif case == "tight_pairs":  # pairs 1e-7 apart: single-child chains ~23 levels deep
        a = rng.uniform(0.0, 1.0, size=(2000, 3))
        pos = np.concatenate([a, a + 1e-7])
    elif case in ("dim1", "dim2"):
        dim = int(case[-1])
        pos = rng.uniform(0.0, 1.0, size=(5000, dim))
    elif case == "box3.7":  # non-dyadic box: the float64 key descent
        box = 3.7
        pos = gen.gen_particles(20_000, 3, clustering=0.7, dim=3, box=box).positions
    elif case == "box0.25":  # dyadic, not 1
        box = 0.25
        pos = gen.gen_particles(20_000, 4, clustering=0.7, dim=3, box=box).positions
    pos = pos.astype(np.float32).astype(np.float64)
    m = rng.uniform(0.5, 1.5, size=len(pos)).astype(np.float32).astype(np.float64)
    return gen.ParticleSet(pos, m, np.zeros_like(pos), box)


@pytest.mark.parametrize("case,bucket", [("n1", 8), ("n8", 8), ("n9", 8), ("coincident", 8), ("tight_pairs", 8),
                                         ("tight_pairs", 1), ("dim1", 8), ("dim2", 8), ("box3.7", 8),
                                         ("box0.25", 32)])
def test_device_build_edge_cases(nb, case, bucket):
    """The bottom-up device build (bb_node_levels / bb_emit_nodes / bb_mass_up)
    on the shapes it special-cases: a root that is a bucket, one particle more
    than a bucket, runs longer than a bucket below the sorted top levels (the
    deep re-sort), deep single-child chains, 1-D / 2-D keys, non-dyadic and
    non-unit dyadic boxes -- equal to the float64 oracle's tree bit for bit."""
    from oracle import oracle as orc
    ps = _edge_set(case)
    a = nb.build_bucket_tree(ps, bucket)
    o = orc.build_bucket_tree(ps.positions, ps.masses, bucket, box=ps.box)
    for k in ("center", "half", "mass", "com", "first_child", "n_child", "pcount"):
        np.testing.assert_array_equal(np.asarray(getattr(a, k)).reshape(np.shape(getattr(o, k))), getattr(o, k),
                                      err_msg=k)
    np.testing.assert_array_equal(a.bucket_ids, o.buckets)
    for b in o.buckets:
        np.testing.assert_array_equal(a.particle_idx(int(b)), o.particle_idx(int(b)))


def test_step_handle_reuse_across_systems(nb):
    """gc_bh_step on ONE handle over systems of different size, clustering and
    box (grow-only device buffers, the sticky sorted key depth, the walk's
    scheduling hints of the previous tree): forces bit-identical to a fresh
    handle's for every system, in every overlap mode."""
    from paper_2008_05712_b200 import _lib as L
    from paper_2008_05712_b200 import generators as gen
    systems = [gen.fp32_exact(gen.gen_plummer(40_000, 3)),  # deep core: the sort depth grows
               gen.fp32_exact(gen.gen_particles(120_000, 4, clustering=0.6, dim=3)),
               gen.fp32_exact(gen.gen_particles(7_000, 5, clustering=0.0, dim=3)),
               gen.fp32_exact(gen.gen_particles(90_000, 6, clustering=0.8, dim=3, box=2.0))]
    for ov in (0, 1, 2):
        st = nb.BHStep(8, 0.7, 1.0, 1e-4)
        L.call("gc_bh_set_overlap", st.handle, ov)
        for rep in range(2):
            for ps in systems:
                got = st(ps.positions, ps.masses, ps.box)
                fresh = nb.BHStep(8, 0.7, 1.0, 1e-4)
                ref = fresh(ps.positions, ps.masses, ps.box)
                np.testing.assert_array_equal(got, ref)


def test_bucket_tree_reset_equals_fresh_build(nb):
    """BucketTree.reset (the distributed backend's per-step rebuild on one
    handle) gives the fresh build's tree for a new set, also after a build
    with forced splits (they are cleared)."""
    from paper_2008_05712_b200 import generators as gen
    a = gen.fp32_exact(gen.gen_particles(60_000, 1, clustering=0.6, dim=3))
    b = gen.fp32_exact(gen.gen_particles(45_000, 2, clustering=0.3, dim=3))
    forced = (np.array([1, 2], np.int32), np.array([[0, 0], [0, 0]], np.uint64))
    t = nb.BucketTree(a, 8, forced=forced)
    t.reset(b)
    f = nb.build_bucket_tree(b, 8)
    for k in ("center", "half", "mass", "com", "first_child", "n_child", "pcount", "pidx"):
        np.testing.assert_array_equal(getattr(t, k), getattr(f, k), err_msg=k)
    np.testing.assert_array_equal(t.bucket_ids, f.bucket_ids)


@pytest.mark.parametrize("bucket,eps,n", [(32, 0.0, 20_000), (1, 1e-4, 5_000), (8, 0.0, 3)])
def test_fused_ring_edge_cases(bucket, eps, n):
    """Opened buckets of 32 particles (33 records from one union entry: the
    ring's largest unit), one-particle buckets, eps = 0 (coincident-source
    guard) and a 3-particle system: fused == staged bit for bit, and both
    within 1e-5 of the oracle."""
    from oracle import oracle as orc
    from paper_2008_05712_b200 import _lib as L
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.fp32_exact(gen.gen_particles(n, 21, clustering=0.8, dim=3))
    tree = nbody.build_bucket_tree(ps, bucket)
    L.call("gc_bh_walk", tree.handle, 0.5)
    res = []
    for mode in (1, 0):
        L.call("gc_bh_set_force_mode", tree.handle, mode)
        f = np.zeros((n, 3))
        L.call("gc_bh_forces", tree.handle, 1.0, eps, L.ptr(f, L.f64p))
        res.append(f)
    np.testing.assert_array_equal(res[0], res[1])
    ot = orc.build_bucket_tree(ps.positions, ps.masses, bucket)
    ol = orc.build_interaction_lists(ot, 0.5)
    ref = orc.eval_forces(ot, ol, ps.positions, ps.masses, 1.0, eps)
    nrm = np.linalg.norm(ref, axis=1)
    err = np.linalg.norm(res[0] - ref, axis=1) / np.where(nrm > 0, nrm, 1.0)
    assert err.max() <= 1e-5


def test_fused_and_staged_reorganisation_bit_identical():
    """The default force path reorganises each force group's sources into
    shared memory inside the force kernel; the staged path writes the same
    runs to HBM first (expand_kernel).  Same records, same order, same
    grouping: the forces and potentials must be bit-identical."""
    from paper_2008_05712_b200 import _lib as L
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.fp32_exact(gen.gen_particles(120_000, 9, clustering=0.6, dim=3))
    tree = nbody.build_bucket_tree(ps, 8)
    L.call("gc_bh_walk", tree.handle, 0.6)
    out = {}
    for mode in (1, 0, 1):
        L.call("gc_bh_set_force_mode", tree.handle, mode)
        n = len(ps.positions)
        f, pot = np.zeros((n, 3)), np.zeros(n)
        L.call("gc_bh_forces_potential", tree.handle, 1.0, 1e-4, L.ptr(f, L.f64p), L.ptr(pot, L.f64p))
        if mode in out:
            np.testing.assert_array_equal(f, out[mode][0])
        out[mode] = (f, pot)
    np.testing.assert_array_equal(out[1][0], out[0][0])
    np.testing.assert_array_equal(out[1][1], out[0][1])


@pytest.mark.parametrize("box", [0.7, 3.3])
def test_inexact_bucket_geometry_lists_bit_exact(box):
    """A box that is not a power of two makes bucket centres / half sizes
    inexact in float32: those buckets skip the float32 certain-accept /
    certain-reject test and take the reference's float64 test for every
    node.  Lists must still equal the oracle's bit for bit."""
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.gen_particles(6000, 17, clustering=0.6, dim=3, box=box)
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, 0.6, ps)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8, box=box)
    ol = orc.build_interaction_lists(ot, 0.6)
    ptr, ids, kind, ic = lists.csr()
    np.testing.assert_array_equal(ptr, ol.ptr)
    np.testing.assert_array_equal(ids, ol.ids)
    np.testing.assert_array_equal(kind, ol.kind)
    np.testing.assert_array_equal(ic, ol.item_count)


def test_pair_stats_bounds():
    """gc_bh_pair_stats: useful interactions <= pairs of target lanes <= issued
    pairs (32 lanes per padded record); gc_bh_sizes' record total matches."""
    from paper_2008_05712_b200 import _lib as L
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.fp32_exact(gen.gen_particles(50_000, 3, clustering=0.6, dim=3))
    tree = nbody.build_bucket_tree(ps, 8)
    L.call("gc_bh_walk", tree.handle, 0.7)
    st = np.zeros(2, np.int64)
    L.call("gc_bh_pair_stats", tree.handle, L.ptr(st, L.i64p))
    inter = nbody.interactions(tree)
    assert 0 < inter <= st[1] <= st[0]
    sz = tree.sizes()
    assert st[0] >= 32 * int(sz[4])  # padded records >= records


def test_overlapped_step_bit_identical():
    """gc_bh_walk_forces_async with the walk/force overlap (programmatic
    dependent launch + readiness queue) gives exactly the forces of the
    back-to-back kernels; so does the one persistent walk+force kernel
    (overlap mode 2) and gc_bh_step."""
    from paper_2008_05712_b200 import _lib as L
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.fp32_exact(gen.gen_particles(150_000, 8, clustering=0.6, dim=3))
    n = len(ps.positions)
    tree = nbody.build_bucket_tree(ps, 8)
    L.call("gc_bh_walk", tree.handle, 0.7)  # stats walk: the overlapped path needs known lists
    out = {}
    for ov in (0, 1, 1, 2, 2):
        L.call("gc_bh_set_overlap", tree.handle, ov)
        L.call("gc_bh_walk_forces_async", tree.handle, 0.7, 1.0, 1e-4)
        f = np.zeros((n, 3))
        L.call("gc_bh_get_forces", tree.handle, L.ptr(f, L.f64p))
        if ov in out:
            np.testing.assert_array_equal(f, out[ov])
        out[ov] = f
    np.testing.assert_array_equal(out[0], out[1])
    np.testing.assert_array_equal(out[0], out[2])
    st = nbody.BHStep(8, 0.7, 1.0, 1e-4)
    g = np.zeros((n, 3))
    for ov in (1, 2, 0):
        L.call("gc_bh_set_overlap", st.handle, ov)
        st(ps.positions, ps.masses, 1.0, g)
        np.testing.assert_array_equal(g, out[0])


@pytest.mark.parametrize("case", ["plummer16k", "clustered1m"])
def test_potential_energy_parity(nb, case):
    """north_star: per-particle forces AND energies within 1e-5 of float64.
    The potential is checked against the oracle's float64 restatement
    (orc_eval_potentials, beside forces_from_points kernels.py:70-88) at
    configs[0] (Plummer 16K) and configs[2] (clustered 1M) full size."""
    from paper_2008_05712_b200 import generators as gen
    from oracle import oracle as orc
    ps = gen.fp32_exact(gen.gen_plummer(16384, 42) if case == "plummer16k"
                        else gen.gen_particles(1_000_000, 42, clustering=0.6, dim=3))
    tree = nb.build_bucket_tree(ps, 8)
    lists = nb.build_interaction_lists(tree, 0.7, ps)
    f, pot = nb.eval_forces_potential(tree, lists, 1.0, 1e-4)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    ol = orc.build_interaction_lists(ot, 0.7)
    ref_f = orc.eval_forces(ot, ol, ps.positions, ps.masses, 1.0, 1e-4)
    ref_p = orc.eval_potentials(ot, ol, ps.positions, ps.masses, 1.0, 1e-4)
    assert rel_err(f, ref_f).max() <= FORCE_RTOL
    ep = np.abs(pot - ref_p) / np.abs(ref_p)
    print(f"{case}: potential rel err median {np.median(ep):.2e} max {ep.max():.2e}")
    assert ep.max() <= FORCE_RTOL


@pytest.mark.parametrize("eps", [1e-7, 1e-12, 0.0])
def test_tiny_softening_finite_and_exact(eps):
    """0 < eps < ~5e-7 makes eps^6 subnormal in float32: the kernels must take
    the cube-of-rsqrt form (finite, coincident sources skipped) and still
    match the oracle.  Includes a duplicated particle."""
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.fp32_exact(gen.gen_particles(6000, 5, clustering=0.6, dim=3))
    pos = ps.positions.copy()
    if eps > 0:
        pos[17] = pos[3]  # coincident pair: needs eps > 0 in the reference
    ps = gen.ParticleSet(pos, ps.masses, np.zeros_like(pos), 1.0)
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, 0.6, ps)
    f, pot = nbody.eval_forces_potential(tree, lists, 1.0, eps)
    assert np.isfinite(f).all() and np.isfinite(pot).all()
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    ol = orc.build_interaction_lists(ot, 0.6)
    ref = orc.eval_forces(ot, ol, ps.positions, ps.masses, 1.0, eps)
    refp = orc.eval_potentials(ot, ol, ps.positions, ps.masses, 1.0, eps)
    assert rel_err(f, ref).max() <= FORCE_RTOL
    assert (np.abs(pot - refp) / np.abs(refp)).max() <= FORCE_RTOL
    f2 = nbody.eval_forces(tree, lists, ps, 1.0, eps)  # force-only instance
    assert rel_err(f2, ref).max() <= FORCE_RTOL


def test_overlap_theta_change_rewalks():
    """Overlap mode with a new theta must not reuse the old theta's pool sizing
    (ADVICE r1): it falls back to the checked walk, forces equal the plain path."""
    from paper_2008_05712_b200 import _lib as L
    from paper_2008_05712_b200 import generators as gen
    from paper_2008_05712_b200 import nbody
    ps = gen.fp32_exact(gen.gen_particles(100_000, 4, clustering=0.6, dim=3))
    n = len(ps.positions)
    tree = nbody.build_bucket_tree(ps, 8)
    L.call("gc_bh_walk", tree.handle, 0.9)
    L.call("gc_bh_set_overlap", tree.handle, 1)
    outs = []
    for th in (0.9, 0.3, 0.3):  # 0.3 needs far more list entries than 0.9
        L.call("gc_bh_walk_forces_async", tree.handle, th, 1.0, 1e-4)
        f = np.zeros((n, 3))
        L.call("gc_bh_get_forces", tree.handle, L.ptr(f, L.f64p))
        outs.append(f)
    L.call("gc_bh_set_overlap", tree.handle, 0)
    L.call("gc_bh_walk_forces_async", tree.handle, 0.3, 1.0, 1e-4)
    f = np.zeros((n, 3))
    L.call("gc_bh_get_forces", tree.handle, L.ptr(f, L.f64p))
    np.testing.assert_array_equal(outs[1], f)
    np.testing.assert_array_equal(outs[2], f)


def test_plummer16m_config4_sampled_parity(nb):
    """configs[3] system (Plummer 16M = 2^24, theta 0.7): the device tree is
    bit-identical to the oracle's (float64 arrays), and on three walk-group
    windows (4096 DFS buckets each, at 10 / 50 / 90 % of the tree) the lists
    are bit-exact and forces + potentials are within 1e-5 of float64."""
    from oracle import oracle as orc
    from paper_2008_05712_b200 import _lib as L
    from paper_2008_05712_b200 import generators as gen
    n = 1 << 24
    ps = gen.fp32_exact(gen.gen_plummer(n, 42))
    tree = nb.build_bucket_tree(ps, 8)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    for k in ("half", "mass", "com", "first_child", "n_child"):
        np.testing.assert_array_equal(getattr(tree, k), getattr(ot, k), err_msg=k)
    np.testing.assert_array_equal(tree.bucket_ids, ot.buckets)
    ngr = np.zeros(1, np.int64)
    L.call("gc_bh_groups", tree.handle, L.ptr(ngr, L.i64p), None)
    wfb = np.zeros(int(ngr[0]) + 1, np.int64)
    L.call("gc_bh_groups", tree.handle, L.ptr(ngr, L.i64p), L.ptr(wfb, L.i64p))
    nbk = len(ot.buckets)
    ntot = 0
    for frac in (0.1, 0.5, 0.9):
        g0 = int(frac * ngr[0])
        g1 = min(int(ngr[0]), g0 + 64)
        b0, b1 = int(wfb[g0]), int(wfb[g1])
        L.call("gc_bh_set_range", tree.handle, g0, g1)
        L.call("gc_bh_walk", tree.handle, 0.7)
        ptr = np.zeros(nbk + 1, np.int64)
        ic = np.zeros(nbk, np.int64)
        L.call("gc_bh_get_lists", tree.handle, L.ptr(ptr, L.i64p), None, None, L.ptr(ic, L.i64p))
        ids = np.zeros(int(ptr[-1]), np.int64)
        kind = np.zeros(int(ptr[-1]), np.int8)
        L.call("gc_bh_get_lists", tree.handle, L.ptr(ptr, L.i64p), L.ptr(ids, L.i64p), L.ptr(kind, L.i8p),
               L.ptr(ic, L.i64p))
        ol = orc.build_interaction_lists(ot, 0.7, bucket_range=(b0, b1))
        np.testing.assert_array_equal(ptr, ol.ptr)
        np.testing.assert_array_equal(ids, ol.ids)
        np.testing.assert_array_equal(kind, ol.kind)
        np.testing.assert_array_equal(ic, ol.item_count)
        f, pot = np.zeros((n, 3)), np.zeros(n)
        L.call("gc_bh_forces_potential", tree.handle, 1.0, 1e-4, L.ptr(f, L.f64p), L.ptr(pot, L.f64p))
        sel = np.concatenate([ot.particle_idx(b) for b in ot.buckets[b0:b1]])
        ref = orc.eval_forces(ot, ol, ps.positions, ps.masses, 1.0, 1e-4, bucket_range=(b0, b1))
        refp = orc.eval_potentials(ot, ol, ps.positions, ps.masses, 1.0, 1e-4, bucket_range=(b0, b1))
        assert rel_err(f[sel], ref[sel]).max() <= FORCE_RTOL
        assert (np.abs(pot[sel] - refp[sel]) / np.abs(refp[sel])).max() <= FORCE_RTOL
        ntot += len(sel)
    L.call("gc_bh_set_range", tree.handle, 0, int(ngr[0]))
    assert ntot > 3 * 4096


def test_periodic_1m_bench_workload_sampled_parity(nb):
    """The bench's periodic workload at full size (configs[2] clustered 1M, 27
    images, theta 0.7): on three 600-bucket ranges the per-bucket entry / item
    counts over all images equal the float64 restatement bit for bit and the
    forces of their particles are within 1e-5."""
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    ps = gen.fp32_exact(gen.gen_particles(1_000_000, 42, clustering=0.6, dim=3))
    tree = nb.build_bucket_tree(ps, 8)
    f, ent, itm = nb.periodic_forces(tree, 0.7, nrep=1)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    nbk = len(ot.buckets)
    for b0 in (0, nbk // 2, nbk - 600):
        b1 = b0 + 600
        fo, eo, io = orc.periodic_forces(ot, ps.positions, ps.masses, 0.7, 1.0, 1, bucket_range=(b0, b1))
        np.testing.assert_array_equal(ent[b0:b1], eo[b0:b1])
        np.testing.assert_array_equal(itm[b0:b1], io[b0:b1])
        pidx = np.concatenate([ot.particle_idx(int(b)) for b in ot.buckets[b0:b1]])
        assert rel_err(f[pidx], fo[pidx]).max() <= FORCE_RTOL


@pytest.mark.parametrize("n,seed,cl,nrep", [(20_000, 5, 0.6, 1), (4096, 9, None, 1), (3000, 2, 0.0, 1), (3000, 2, 0.0, 0)])
def test_periodic_walk_matches_oracle(nb, n, seed, cl, nrep):
    """Periodic BH (no reference implementation -- the float64
    restatement oracle/gcharm_oracle.c orc_periodic_forces): per-bucket entry
    and item counts over all (2 nrep + 1)^3 images bit-exact (every opening
    decision, shifted centres of mass), forces within 1e-5 per particle; the
    open-boundary path is untouched afterwards."""
    from oracle import oracle as orc
    from paper_2008_05712_b200 import generators as gen
    ps = gen.fp32_exact(gen.gen_plummer(n, seed) if cl is None else gen.gen_particles(n, seed, cl, 3))
    tree = nb.build_bucket_tree(ps, 8)
    f, ent, itm = nb.periodic_forces(tree, 0.7, nrep=nrep)
    ot = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    fo, eo, io = orc.periodic_forces(ot, ps.positions, ps.masses, 0.7, 1.0, nrep)
    np.testing.assert_array_equal(ent, eo)
    np.testing.assert_array_equal(itm, io)
    assert rel_err(f, fo).max() <= FORCE_RTOL
    lists = nb.build_interaction_lists(tree, 0.7, ps)
    ol = orc.build_interaction_lists(ot, 0.7)
    ptr, ids, kind, ic = lists.csr()
    np.testing.assert_array_equal(ids, ol.ids)
    assert rel_err(nb.eval_forces(tree, lists, ps), orc.eval_forces(ot, ol, ps.positions, ps.masses)).max() <= FORCE_RTOL
    with pytest.raises(ValueError):
        nb.periodic_forces(tree, 0.7, nrep=2)  # 125 images exceed the entry's image tag

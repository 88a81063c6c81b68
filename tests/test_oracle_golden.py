"""Pin the CPU oracle (oracle/) against the reference's own outputs.

Fixtures come from tests/golden/make_golden.py, which ran the reference
(hetero-rt) in the dev container.  Bit-exact equality for trees, lists and
float64 forces; these tests need no GPU.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import dm as odm
from oracle import oracle as orc

from conftest import GOLDEN


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


CASES = [("nbody2d_300", [0.0, 0.3, 0.7], 0.7), ("nbody3d_2048", [0.0, 0.7], 0.7),
         ("plummer3d_4096", [0.7], 0.7)]


def tag(th):
    return f"theta{th:g}".replace(".", "p")


@pytest.mark.parametrize("name,thetas,ftheta", CASES)
def test_tree_lists_forces_bit_exact(name, thetas, ftheta):
    g = load(name)
    t = orc.build_bucket_tree(g["positions"], g["masses"], int(g["bucket_size"]), float(g["box"]))
    for k in ("center", "half", "mass", "com", "first_child", "n_child", "buckets", "pidx"):
        np.testing.assert_array_equal(getattr(t, k), g[f"tree_{k}"], err_msg=k)
    pc = np.where(t.first_child < 0, t.pcount, 0)
    np.testing.assert_array_equal(pc, g["tree_pcount"])
    for th in thetas:
        L = orc.build_interaction_lists(t, th)
        for k in ("ptr", "ids", "kind", "item_count"):
            np.testing.assert_array_equal(getattr(L, k), g[f"lists_{tag(th)}_{k}"], err_msg=f"{th} {k}")
        if th == ftheta:
            f = orc.eval_forces(t, L, g["positions"], g["masses"])
            np.testing.assert_array_equal(f, g[f"forces_{tag(th)}"])


def test_plummer16k_digests():
    """Config 1 (Plummer 16K, theta 0.7): tree, lists, float64 forces equal the
    reference's bit for bit (sha256 over the exact arrays)."""
    from paper_2008_05712_b200 import generators as gen
    d = json.load(open(os.path.join(GOLDEN, "digests.json")))["digests"]["plummer3d_16384"]
    ps = gen.fp32_exact(gen.gen_plummer(16384, 42))
    t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    pc = np.where(t.first_child < 0, t.pcount, 0)
    assert sha(t.center, t.half, t.mass, t.com, t.first_child, t.n_child, pc, t.buckets, t.pidx) == d["tree"]
    L = orc.build_interaction_lists(t, 0.7)
    assert sha(L.ptr, L.ids, L.kind, L.item_count) == d["lists_theta0p7"]
    f = orc.eval_forces(t, L, ps.positions, ps.masses)
    assert sha(f) == d["forces_theta0p7"]


def test_kernels_golden():
    g = load("kernels")
    np.testing.assert_array_equal(orc.forces_from_points(g["ppos"], g["pmass"], g["spos"], g["smass"], 1.0, 1e-4),
                                  g["ffp"])
    np.testing.assert_array_equal(orc.forces_from_points(g["ppos"], g["pmass"], g["spos"], g["smass"], 1.0, 0.0),
                                  g["ffp_eps0"])
    fa, fb = orc.md_cross_forces(g["md_a"], g["md_b"], 1.0, 25.0)
    np.testing.assert_array_equal(fa, g["md_fa"])
    np.testing.assert_array_equal(fb, g["md_fb"])
    np.testing.assert_array_equal(orc.md_self_forces(g["md_self_pos"], 1.0, 25.0), g["md_self_f"])
    np.testing.assert_array_equal(orc.direct_forces(g["direct_pos"], g["direct_mass"], 1.0, 1e-4), g["direct_f"])
    off = np.concatenate([[0], np.cumsum(g["runs_lens"])])
    for i in range(len(g["runs_lens"])):
        a = g["runs_in"][off[i]:off[i + 1]]
        assert orc.count_address_runs(a) == g["runs_out"][i]
        assert odm.count_runs(a.tolist()) == g["runs_out"][i]


@pytest.mark.parametrize("tagname,periodic", [("wall", False), ("per", True)])
def test_md2d_golden(tagname, periodic):
    g = load("md2d")
    f = orc.md2d_compute_forces(g[f"{tagname}_pos0"], g[f"{tagname}_patch0"], 10, 10, 1.0, 1.0, 25.0, periodic)
    np.testing.assert_array_equal(f, g[f"{tagname}_f0"])
    pos, vel, patch = g[f"{tagname}_pos0"], g[f"{tagname}_vel0"], g[f"{tagname}_patch0"]
    for _ in range(3):
        pos, vel, patch = orc.md2d_step(pos, vel, patch, 10, 10, 1.0, 1.0, 0.08, 25.0, periodic)
    np.testing.assert_array_equal(pos, g[f"{tagname}_pos3"])
    np.testing.assert_array_equal(vel, g[f"{tagname}_vel3"])
    np.testing.assert_array_equal(patch, g[f"{tagname}_patch3"])


def test_dm_plans_golden():
    cases = json.load(open(os.path.join(GOLDEN, "dm_plans.json")))
    for c in cases:
        mem = odm.OracleDM(c["cap"], c["slot"], c["mode"])
        for (members, now), want in zip(c["batches"], c["result"]):
            try:
                p = mem.plan(members, now)
            except odm.OracleCapacityError:
                assert not want["ok"], c["name"]
                continue
            assert want["ok"], c["name"]
            assert p["to_transfer"] == want["to_transfer"], c["name"]
            assert p["addresses"] == want["addresses"], c["name"]
            assert p["bounds"] == want["bounds"]
            assert p["total_bytes"] == want["total_bytes"]
            assert p["indirection_bytes"] == want["indirection_bytes"]
            assert odm.member_transactions(p) == want["transactions"]
            if c["mode"] != "redundant":
                assert sorted(mem.slot_of.items()) == [tuple(x) for x in want["table"]]
            if c["release"]:
                mem.release(members)


def test_aggregator_golden():
    g = json.load(open(os.path.join(GOLDEN, "aggregator.json")))
    for e in g["emissions"]:
        arr = [tuple(a) for a in e["arrivals"]]
        got = odm.emissions(arr, e["max_size"], e["polls"])
        assert [[t, list(ids)] for t, ids in got] == e["emissions"]
    for p in g["partitions"]:
        assert odm.partition(p["items"], p["share"], p["nearest"]) == p["cut"]


def _direct_potential(pos, mass, g, eps):
    """Independent numpy float64 direct sum -g m_i sum_{j: x_j != x_i} m_j / sqrt(r^2 + eps^2)."""
    d = pos[None, :, :] - pos[:, None, :]
    r2 = eps * eps + (d * d).sum(axis=2)
    same = np.all(d == 0.0, axis=2)
    w = np.where(same, 0.0, mass[None, :] / np.sqrt(r2))
    return -g * mass * w.sum(axis=1)


@pytest.mark.parametrize("name,dim", [("nbody2d_300", 2), ("nbody3d_2048", 3)])
def test_potential_oracle_pinned_by_direct_sum(name, dim):
    """The BH potential restatement (no reference counterpart) is pinned by a
    known answer: at theta = 0 every list is opened particles only, so the
    list potential equals the direct sum (up to summation order)."""
    g = load(name)
    pos, m = g["positions"], g["masses"]
    t = orc.build_bucket_tree(pos, m, int(g["bucket_size"]), box=float(g["box"]))
    ol = orc.build_interaction_lists(t, 0.0)
    phi = orc.eval_potentials(t, ol, pos, m, 1.0, 1e-4)
    ref = _direct_potential(pos, m, 1.0, 1e-4)
    np.testing.assert_allclose(phi, ref, rtol=1e-12)
    # theta > 0: monopole approximation, within the acceptance-10 tolerance scale
    ol7 = orc.build_interaction_lists(t, 0.7)
    phi7 = orc.eval_potentials(t, ol7, pos, m, 1.0, 1e-4)
    assert np.median(np.abs(phi7 - ref) / np.abs(ref)) < 4e-3


def test_potential_oracle_coincident_skip():
    """Coincident sources are skipped exactly as in forces_from_points (kernels.py:78-84)."""
    pos = np.array([[0.25, 0.25, 0.25], [0.25, 0.25, 0.25], [0.75, 0.25, 0.25]])
    m = np.array([1.0, 2.0, 3.0])
    t = orc.build_bucket_tree(pos, m, 8)
    ol = orc.build_interaction_lists(t, 0.5)
    phi = orc.eval_potentials(t, ol, pos, m, 1.0, 0.0)
    np.testing.assert_allclose(phi, [-1.0 * 3.0 / 0.5, -2.0 * 3.0 / 0.5, -3.0 * 3.0 / 0.5], rtol=1e-15)


def test_lj3d_multicore_baseline_matches_serial():
    """The multi-core LJ restatement (the CPU baseline's form) evaluates the
    same pairs as the serial parity restatement: equal to rounding."""
    from paper_2008_05712_b200.generators import gen_lj_fcc
    s = gen_lj_fcc(8)
    d = (s.cells,) * 3
    f1, e1 = orc.lj3d_compute_forces(s.positions, d, s.cell_size, nthreads=1)
    f2, e2 = orc.lj3d_compute_forces(s.positions, d, s.cell_size, nthreads=4)
    np.testing.assert_allclose(f2, f1, rtol=0, atol=1e-11)
    np.testing.assert_allclose(e2, e1, rtol=0, atol=1e-11)


def test_periodic_oracle_pinned():
    """The periodic BH restatement (no reference implementation): nrep = 0 is
    the open-boundary eval_forces bit for bit, and at theta = 0 (every node
    opened) it equals an independent numpy direct sum over the 27 images."""
    from paper_2008_05712_b200 import generators as gen
    ps = gen.fp32_exact(gen.gen_particles(600, 4, clustering=0.5, dim=3))
    t = orc.build_bucket_tree(ps.positions, ps.masses, 8)
    f0, _, i0 = orc.periodic_forces(t, ps.positions, ps.masses, 0.7, 1.0, 0)
    lists = orc.build_interaction_lists(t, 0.7)
    np.testing.assert_array_equal(f0, orc.eval_forces(t, lists, ps.positions, ps.masses))
    np.testing.assert_array_equal(i0, lists.item_count)
    f, _, _ = orc.periodic_forces(t, ps.positions, ps.masses, 0.0, 1.0, 1)
    p, m, eps = ps.positions, ps.masses, 1e-4
    ref = np.zeros_like(p)
    for ix in (-1, 0, 1):
        for iy in (-1, 0, 1):
            for iz in (-1, 0, 1):
                q = p + np.array([ix, iy, iz], float)
                d = q[None, :, :] - p[:, None, :]
                r2 = eps * eps + (d * d).sum(axis=2)
                same = np.all(d == 0.0, axis=2)
                w = np.where(same, 0.0, m[None, :] / (r2 * np.sqrt(r2)))
                ref += m[:, None] * (d * w[:, :, None]).sum(axis=1)
    np.testing.assert_allclose(f, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())

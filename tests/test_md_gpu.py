"""GPU parity of the cell-pair MD path.

2-D soft repulsion (the reference's MD, hr/workloads/md.py) against the
reference's golden forces/steps; 3-D Lennard-Jones (no reference; parity
unpinned) against the float64 oracle restatement and an independent O(n^2)
minimum-image brute force.  Both paths compute in float64 with the reference's
cutoff decisions; tolerances are per particle ||dF|| / ||F|| <= FORCE_RTOL
(particles with no neighbours must be exactly zero).
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

FORCE_RTOL = 1e-10


def rel_err(a, b):
    na = np.linalg.norm(b, axis=1)
    d = np.linalg.norm(a - b, axis=1)
    zero = na == 0
    assert np.all(d[zero] == 0)
    return (d[~zero] / na[~zero]) if (~zero).any() else np.zeros(1)


@pytest.fixture(scope="module")
def md():
    from paper_2008_05712_b200 import md
    return md


def grid_from(md, g, tag, k):
    return md.PatchGrid(10, 10, 1.0, 1.0, g[f"{tag}_pos{k}"].copy(), g[f"{tag}_vel{k}"].copy(),
                        g[f"{tag}_patch{k}"].copy())


@pytest.mark.parametrize("tag,periodic", [("wall", False), ("per", True)])
def test_md2d_golden_forces_and_steps(md, tag, periodic):
    g = np.load(os.path.join(GOLDEN, "md2d.npz"))
    grid = grid_from(md, g, tag, 0)
    f = md.compute_forces(grid, 25.0, periodic)
    assert rel_err(f, g[f"{tag}_f0"]).max() <= FORCE_RTOL
    for _ in range(3):
        md.md_step(grid, 0.08, 25.0, periodic)
    np.testing.assert_allclose(grid.positions, g[f"{tag}_pos3"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(grid.velocities, g[f"{tag}_vel3"], rtol=0, atol=1e-8)
    np.testing.assert_array_equal(grid.patch_of, g[f"{tag}_patch3"])
    f3 = md.compute_forces(grid, 25.0, periodic)
    assert rel_err(f3, g[f"{tag}_f3"]).max() <= 1e-6  # trajectories agree to ~1e-12


def test_md2d_reference_properties(md):
    # migration containment (test_workloads.py:172-181)
    grid, _ = md.gen_md_system((3, 3), 10, cutoff=1.0, seed=22)
    before = grid.patch_of.copy()
    for _ in range(5):
        md.md_step(grid, dt=0.3)
    assert (grid.patch_of != before).any()
    r = (grid.positions[:, 0] // grid.patch_size).astype(int).clip(0, 2)
    c = (grid.positions[:, 1] // grid.patch_size).astype(int).clip(0, 2)
    np.testing.assert_array_equal(grid.patch_of, r * 3 + c)
    # zero velocity, isolated particles: fixed point (183-188)
    grid, _ = md.gen_md_system((2, 2), 1, cutoff=1.0, seed=23)
    grid.velocities[:] = 0.0
    before = grid.patch_of.copy()
    md.md_step(grid, dt=0.1)
    np.testing.assert_array_equal(grid.patch_of, before)
    # conservation over 100 steps, positions inside the walls (190-197)
    grid, _ = md.gen_md_system((4, 4), 6, cutoff=1.0, seed=24)
    n = len(grid.positions)
    for _ in range(100):
        md.md_step(grid, dt=0.2)
    assert grid.populations().sum() == n
    assert ((grid.positions >= 0) & (grid.positions <= np.array(grid.box))).all()
    # periodic wrap (247-253)
    grid, _ = md.gen_md_system((4, 4), 6, cutoff=1.0, seed=31)
    for _ in range(30):
        md.md_step(grid, dt=0.3, periodic=True)
    assert grid.populations().sum() == n
    assert ((grid.positions >= 0) & (grid.positions < np.array(grid.box))).all()
    # Newton's third law: forces sum to zero
    grid, _ = md.gen_md_system((6, 6), 20, cutoff=1.0, seed=5)
    f = md.compute_forces(grid)
    assert np.abs(f.sum(axis=0)).max() <= 1e-9 * np.abs(f).max()


def test_md2d_67x67_digest_scale(md):
    """The reference's 67x67x24 analogue (107,736 atoms): forces equal the
    oracle restatement (itself bit-equal to the reference, digests.json)."""
    from oracle import oracle as orc
    grid, _ = md.gen_md_system((67, 67), 24, 1.0, 7)
    f = md.compute_forces(grid)
    ref = orc.md2d_compute_forces(grid.positions, grid.patch_of, 67, 67, 1.0, 1.0, 25.0, False)
    assert rel_err(f, ref).max() <= FORCE_RTOL


def jitter(s, seed=0, amp=0.03):
    """Thermal-like displacement of the perfect lattice (whose net forces are
    ~1e-5 by symmetry and make relative errors meaningless)."""
    rng = np.random.default_rng(seed)
    box = s.cells * s.cell_size
    p = s.positions + rng.normal(0.0, amp, size=s.positions.shape)
    s.positions = np.remainder(p.astype(np.float32).astype(np.float64), box)
    return s


def small_lj():
    from paper_2008_05712_b200.generators import gen_lj_fcc
    return jitter(gen_lj_fcc(lattice_cells=6, seed=3))


def test_lj_small_vs_oracle_and_bruteforce(md):
    from oracle import oracle as orc
    s = small_lj()
    sysd = md.LJSystem(s)
    f, e = sysd.forces()
    dims = (s.cells,) * 3
    fo, eo = orc.lj3d_compute_forces(s.positions, dims, s.cell_size, s.rc, s.eps, s.sigma, True)
    assert rel_err(f, fo).max() <= FORCE_RTOL
    np.testing.assert_allclose(e, eo, rtol=1e-10, atol=1e-12)
    box = np.array(dims) * s.cell_size
    fb, eb = orc.lj3d_bruteforce(s.positions, box, s.rc, s.eps, s.sigma, True)
    assert rel_err(f, fb).max() <= 1e-9
    assert np.abs(f.sum(axis=0)).max() <= 1e-9 * np.abs(f).max()


def test_lj_steps_vs_oracle(md):
    from oracle import oracle as orc
    s = small_lj()
    sysd = md.LJSystem(s)
    sysd.run(10)
    p, v, _ = sysd.state()
    pos, vel = s.positions.copy(), s.velocities.copy()
    dims = (s.cells,) * 3
    for _ in range(10):
        pos, vel, _, _ = orc.lj3d_step(pos, vel, dims, s.cell_size, s.dt, s.rc, s.eps, s.sigma)
    np.testing.assert_allclose(p, pos, rtol=0, atol=1e-9)
    np.testing.assert_allclose(v, vel, rtol=0, atol=1e-8)


def test_lj_108k_config2_forces(md):
    """configs[1]: FCC 30^3 x 4 = 108,000 atoms, rc 2.5, 20^3 cells."""
    from oracle import oracle as orc
    from paper_2008_05712_b200.generators import gen_lj_fcc
    s = jitter(gen_lj_fcc(30), seed=1)
    assert s.positions.shape[0] == 108000 and s.cells == 20
    sysd = md.LJSystem(s)
    f, e = sysd.forces()
    fo, eo = orc.lj3d_compute_forces(s.positions, (20, 20, 20), s.cell_size, s.rc, s.eps, s.sigma, True)
    assert rel_err(f, fo).max() <= FORCE_RTOL
    np.testing.assert_allclose(e, eo, rtol=1e-10, atol=1e-12)
    # 100 steps: momentum stays ~0, energy bounded (symplectic)
    e0 = 0.5 * (s.velocities ** 2).sum() + eo.sum()
    sysd.run(100)
    p, v, _ = sysd.state()
    f2, e2 = sysd.forces()
    e1 = 0.5 * (v ** 2).sum() + e2.sum()
    assert abs(e1 - e0) / abs(e0) < 2e-2
    assert np.abs(v.sum(axis=0)).max() < 1e-6 * len(v)


def test_lj_8m_config5_forces(md):
    """configs[4] system at full size: FCC 126^3 x 4 = 8,001,504 atoms, 84^3
    cells -- every atom's force and energy against the float64 oracle (the
    system bench.py times as configs[4] on one GPU)."""
    from oracle import oracle as orc
    from paper_2008_05712_b200.generators import gen_lj_fcc
    s = jitter(gen_lj_fcc(126), seed=5)
    assert s.positions.shape[0] == 8_001_504 and s.cells == 84
    sysd = md.LJSystem(s)
    f, e = sysd.forces()
    fo, eo = orc.lj3d_compute_forces(s.positions, (84, 84, 84), s.cell_size, s.rc, s.eps, s.sigma, True)
    assert rel_err(f, fo).max() <= FORCE_RTOL
    np.testing.assert_allclose(e, eo, rtol=1e-10, atol=1e-12)


def test_lj_column_phase_varying_rate(md):
    """configs[4]'s force work arriving at a varying generation rate: column
    requests (arrival = ready_cost x largest neighbour-cell population +
    lognormal lulls) combined by the device trigger into batches of at most
    max_size, each one column-kernel launch -- forces and energies bit-identical
    to the whole-system launch; the batches are the host poll_combine's."""
    from paper_2008_05712_b200.aggregator import AggregatorState, observe_arrival, poll_combine
    from paper_2008_05712_b200.generators import gen_lj_fcc
    from paper_2008_05712_b200.runtime import WorkRequest
    s = jitter(gen_lj_fcc(30), seed=4)
    sysd = md.LJSystem(s)
    f0, e0 = sysd.forces()
    ph = md.LJColumnPhase(sysd, max_size=300, ready_cost=0.01, pieces=8, piece_gap=4.0, tick=0.25)
    f1, e1, batches, ms = ph.run()
    np.testing.assert_array_equal(f1, f0)
    np.testing.assert_array_equal(e1, e0)
    assert sum(c for _, c, _ in batches) == ph.ncol and ms > 0
    order, t = ph.arrivals(sysd.state()[0])
    ev_t, ev_p = ph.events(t)
    st = AggregatorState("md", 300, 2.0)
    ref = []
    i = 0
    for ti, pi in zip(ev_t, ev_p):
        if not pi:  # an arrival (else a timeline tick: a poll only)
            st.pending.append(WorkRequest(i, 0, "md", [], 1, ti, 0))
            observe_arrival(st, ti)
            i += 1
        while (c := poll_combine(st, ti)) is not None:
            ref.append((c.members[0].id, len(c.members)))
    k = sum(n for _, n in ref)
    while k < len(t):
        ref.append((k, min(300, len(t) - k)))
        k += ref[-1][1]
    assert [(a, c) for a, c, _ in batches] == ref
    assert any(c < 300 for _, c, _ in batches[:-1])  # the lulls fire timeout flushes

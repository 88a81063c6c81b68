"""Ewald kernel class on the device (csrc/ewald.cuh) against the float64
oracle restatement (itself pinned by known answers, test_ewald_cpu.py):
moments, the correction at arbitrary points, and the class run through the
runtime API next to the force class (executor.py, NBodyParams(ewald=True),
hr/workloads/nbody.py:317-323).  Tolerances: max |delta| / max |value|
<= 1e-12 (float64, different summation order)."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-12
TIGHT = dict(alpha=2.0, nrep=4, ewcut=3.5, hcut=4.5)


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def test_moments_and_points_match_oracle():
    from paper_2008_05712_b200 import ewald
    rng = np.random.default_rng(5)
    src = 0.5 + 0.1 * rng.standard_normal((3000, 3))
    m = rng.uniform(0.5, 1.5, 3000)
    mom = ewald.multipole_moments(src, m)
    want = orc.ewald_moments(src, m)
    assert rel(mom[:4], want[:4]) <= 1e-14
    assert rel(mom[4:], want[4:]) <= 1e-12
    x = rng.random((257, 3))
    for p in (ewald.EwaldParams(), ewald.EwaldParams(**TIGHT), ewald.EwaldParams(alpha=2.6, nrep=3, ewcut=2.9,
                                                                                 hcut=6.0)):
        a, phi = ewald.ewald_correction(x, want, p)
        kw = dict(L=p.L, alpha=p.alpha, nrep=p.nrep, ewcut=p.ewcut, hcut=p.hcut)
        ao, po = orc.ewald_correction(x, want, **kw)
        assert rel(a, ao) <= TOL
        assert rel(phi, po) <= TOL


def test_device_symmetry_zero_and_near_field():
    from paper_2008_05712_b200 import ewald
    mom = np.array([1.0, 0.3, 0.4, 0.5, 0, 0, 0, 0, 0, 0])
    x = np.array([[0.8, 0.4, 0.5], [0.8, 0.9, 1.0], [0.3, 0.4, 0.5]])  # half-box points and the mass itself
    a, _ = ewald.ewald_correction(x, mom, ewald.EwaldParams(**TIGHT))
    d = x[:2] - mom[1:4]
    direct = -d / np.linalg.norm(d, axis=1)[:, None] ** 3
    np.testing.assert_allclose(a[:2] + direct, 0.0, atol=1e-12)
    np.testing.assert_allclose(a[2], 0.0, atol=1e-12)  # central replica's series branch at r = 0


def test_ewald_class_through_runtime():
    from paper_2008_05712_b200 import ewald, generators as gen, nbody
    from paper_2008_05712_b200.executor import GpuForceExecutor
    from paper_2008_05712_b200.memory import MemoryMode
    ps = gen.fp32_exact(gen.gen_particles(4000, 13, clustering=0.6, dim=3))
    tree = nbody.build_bucket_tree(ps, 8)
    lists = nbody.build_interaction_lists(tree, 0.6, ps)
    base = GpuForceExecutor(tree, lists, MemoryMode.REUSE_SORTED, capacity_bytes=16 << 20, max_size=64).run()
    p = ewald.EwaldParams()
    ex = GpuForceExecutor(tree, lists, MemoryMode.REUSE_SORTED, capacity_bytes=32 << 20, max_size=64, ewald=p,
                          ewald_max_size=96)
    res = ex.run()
    nb = len(ex.ptr) - 1
    assert ex.runtime.completed_count == 2 * nb and ex.runtime.pending_count == 0
    ew = [b for b in res.batches if b.kernel_class == "ewald"]
    assert sum(b.members for b in ew) == nb and max(b.members for b in ew) <= 96
    assert all(b.positions == b.members for b in ew)  # one buffer per ewald request
    np.testing.assert_array_equal(res.forces, base.forces)  # the force class is unchanged
    mom = ewald.tree_moments(tree)
    want = orc.ewald_moments(ps.positions, ps.masses)
    assert rel(mom, want) <= 1e-12
    acc, pot = orc.ewald_correction(ps.positions, mom)
    np.testing.assert_array_less(-1, res.ewald_pot)  # finite
    assert rel(res.ewald_forces, ps.masses[:, None] * acc) <= TOL
    assert rel(res.ewald_pot, ps.masses * pot) <= TOL


def test_ewald_kernel_spec_and_max_size():
    from paper_2008_05712_b200.aggregator import compute_max_size
    from paper_2008_05712_b200.devicesim import b200_device_spec, b200_kernel_spec
    k = b200_kernel_spec("ewald_member")
    assert k.threads_per_block == 256 and k.registers_per_thread > 64
    assert compute_max_size(k, b200_device_spec()) >= 148

"""Multi-GPU MD (x-slab decomposition) on ONE device: K slabs
of one periodic LJ system exchanged in-process must reproduce the whole-domain
run bit for bit (same kernels, global image shifts, cells ordered by global id)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def system():
    from paper_2008_05712_b200.generators import gen_lj_fcc
    return gen_lj_fcc(10, repeat_x=4)  # 16,000 atoms, 24 x 6 x 6 cells


@pytest.fixture(scope="module")
def whole(system):
    from paper_2008_05712_b200 import md
    s = md.LJSystem(system)
    s.run(5)
    p, v, _ = s.state()
    return p, v


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_slabs_match_whole_domain(system, whole, k):
    from paper_2008_05712_b200 import md_dist
    p, v = md_dist.run_local(system, k, 5)
    np.testing.assert_array_equal(p, whole[0])
    np.testing.assert_array_equal(v, whole[1])


def test_slab_forces_match_whole_domain(system):
    """One slab step's integrator consumed bit-identical forces: compare the
    first-step velocities of a 3-slab run with the whole-domain step."""
    from paper_2008_05712_b200 import md, md_dist
    s = md.LJSystem(system)
    s.run(1)
    p1, v1, _ = s.state()
    p, v = md_dist.run_local(system, 3, 1)
    np.testing.assert_array_equal(v, v1)
    np.testing.assert_array_equal(p, p1)


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_device_count_slabs_match_whole_domain(system, whole, k):
    """The device-count step (fixed-capacity messages, counts on the device,
    no host round trip inside a step) is bit-identical to the whole domain."""
    from paper_2008_05712_b200 import md_dist
    p, v = md_dist.run_local_dev(system, k, 5)
    np.testing.assert_array_equal(p, whole[0])
    np.testing.assert_array_equal(v, whole[1])


def test_device_count_step_has_no_host_sync():
    """LJSlab.step_dev's source issues no device synchronisation or host read
    of a device value (the per-step path of §8e)."""
    import inspect

    from paper_2008_05712_b200 import md_dist
    for fn in (md_dist.LJSlab.step_dev, md_dist.LJSlab.pack_dev, md_dist.LJSlab.exchange_dev,
               md_dist.LJSlab.set_halo_dev, md_dist.LJSlab.advance_dev, md_dist.LJSlab.take_migrants_dev,
               md_dist.DistTransport.exchange_fixed):
        src = inspect.getsource(fn)
        for bad in (".item()", "synchronize", ".cpu()", ".tolist()", "numpy()"):
            assert bad not in src, (fn.__name__, bad)

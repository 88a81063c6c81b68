"""Device closed-loop MD (csrc/md_loop.cu) against the reference's recorded
MDWorkload runs: the final grid bit for bit (float64, numba loop order), the
per-step work requests / "interact" messages / completions, and the
runtime's invocation totals per entry method."""
import numpy as np
import pytest

from test_mdloop_cpu import CASES, golden, params

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag", CASES)
def test_device_closed_loop_bit_exact(tag):
    from paper_2008_05712_b200.md import MDWorkload
    g = golden()
    p = params(g, tag)
    wl = MDWorkload(p)
    res = wl.run()
    np.testing.assert_array_equal(wl.grid.positions, g[f"{tag}_pos"])
    np.testing.assert_array_equal(wl.grid.velocities, g[f"{tag}_vel"])
    np.testing.assert_array_equal(wl.grid.patch_of, g[f"{tag}_patch"])
    np.testing.assert_array_equal(res.work_requests, g[f"{tag}_tasks"])
    np.testing.assert_array_equal(res.interact_messages, g[f"{tag}_inputs"])
    np.testing.assert_array_equal(res.completions, g[f"{tag}_tasks"])
    assert res.invocations == {"interact": int(g[f"{tag}_inv_interact"]),
                               "work_done": int(g[f"{tag}_inv_work_done"]),
                               "step_barrier": int(g[f"{tag}_inv_barrier"])}
    assert wl.step == p.steps


def test_device_closed_loop_scale_and_rerun():
    """67 x 67 x 24 (107,736 atoms, the reference's large MD analogue): the
    device loop equals the oracle's step sequence bit for bit, and a rerun
    from the same start is identical (deterministic despite the dynamic
    ready queue)."""
    from oracle import oracle as orc
    from paper_2008_05712_b200.md import MDParams, MDWorkload
    p = MDParams(rows=67, cols=67, steps=4, dt=0.05)
    wl = MDWorkload(p)
    pos, vel, patch = wl.grid.positions.copy(), wl.grid.velocities.copy(), wl.grid.patch_of.copy()
    r1 = wl.run()
    a = (wl.grid.positions.copy(), wl.grid.velocities.copy(), wl.grid.patch_of.copy())
    for _ in range(p.steps - 1):
        pos, vel, patch = orc.md2d_step(pos, vel, patch, 67, 67, 1.0, 1.0, p.dt, p.stiffness, False)
    np.testing.assert_array_equal(a[0], pos)
    np.testing.assert_array_equal(a[1], vel)
    np.testing.assert_array_equal(a[2], patch)
    wl2 = MDWorkload(p)
    r2 = wl2.run()
    np.testing.assert_array_equal(wl2.grid.positions, a[0])
    np.testing.assert_array_equal(r1.work_requests, r2.work_requests)
    from paper_2008_05712_b200.md import neighbor_pairs
    # compute_forces segments without walls: self + in-grid half-shell neighbours
    nseg = sum(1 + sum(0 <= r + dr < 67 and 0 <= c + dc < 67 for dr, dc in ((0, 1), (1, -1), (1, 0), (1, 1)))
               for r in range(67) for c in range(67))
    assert wl.topology() == (67 * 67, len(neighbor_pairs(67, 67)), nseg)

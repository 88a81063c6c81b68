"""Closed-loop MD (hr/workloads/md.py MDWorkload through hr/timeline.py):
the oracle restatement and the host mirrors against the reference's recorded
runs (tests/golden/mdloop.npz, made by tests/golden/make_mdloop_golden.py).

The oracle replays the loop -- `steps` rounds of pair_work, steps - 1
md_step updates -- and must land on the reference's final grid bit for bit;
the per-step work-request / message counts follow from neighbor_pairs and
the populations (md.py:82-89, 232-253)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

CASES = ["wall", "per", "tiny", "strip", "sparse"]


def golden():
    return np.load(os.path.join(GOLDEN, "mdloop.npz"))


def params(g, tag):
    from paper_2008_05712_b200.md import MDParams
    kw = {}
    for f in MDParams.__dataclass_fields__:
        v = g[f"{tag}_param_{f}"]
        kw[f] = v.item()
    return MDParams(**kw)


@pytest.mark.parametrize("tag", CASES)
def test_oracle_closed_loop_matches_reference(tag):
    from oracle import oracle as orc
    from paper_2008_05712_b200 import md
    g = golden()
    p = params(g, tag)
    grid, _ = md.gen_md_system((p.rows, p.cols), p.particles_per_patch, p.cutoff, p.seed)
    pos, vel, patch = grid.positions, grid.velocities, grid.patch_of
    tasks, inputs = [], []
    for k in range(p.steps):
        grid.patch_of = patch
        work = md.pair_work(grid, p.periodic)
        tasks.append(len(work))
        inputs.append(sum(1 if a == b else 2 for a, b, _ in work))
        if k + 1 < p.steps:
            pos, vel, patch = orc.md2d_step(pos, vel, patch, p.rows, p.cols, grid.patch_size, p.cutoff, p.dt,
                                            p.stiffness, p.periodic)
    np.testing.assert_array_equal(pos, g[f"{tag}_pos"])
    np.testing.assert_array_equal(vel, g[f"{tag}_vel"])
    np.testing.assert_array_equal(patch, g[f"{tag}_patch"])
    np.testing.assert_array_equal(tasks, g[f"{tag}_tasks"])
    np.testing.assert_array_equal(inputs, g[f"{tag}_inputs"])
    assert int(g[f"{tag}_inv_interact"]) == sum(tasks) == int(g[f"{tag}_inv_work_done"])
    assert int(g[f"{tag}_msg_interact"]) == sum(inputs)
    assert int(g[f"{tag}_inv_barrier"]) == p.steps


def test_mdparams_mirror_defaults():
    import dataclasses
    from paper_2008_05712_b200.md import MDParams
    g = golden()
    assert dataclasses.asdict(MDParams()) == dataclasses.asdict(params(g, "wall"))

"""Golden closed-loop MD runs of the REFERENCE (hr/workloads/md.py MDWorkload
driven by hr/timeline.py's message-driven runtime), for the device closed loop
(tests/test_mdloop_*.py).  Dev container only:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_mdloop_golden.py

Per case it stores the grid after the run (positions, velocities, patch_of),
the per-step work-request counts and "interact" messages the workload
scheduled (_begin_step, md.py:232-253), and the runtime's invocation counts
per entry method (runtime.py:95-118).
"""
import dataclasses
import os
import sys

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from hetero_rt import kernels as rk  # noqa: E402
from hetero_rt.config import ExperimentConfig  # noqa: E402
from hetero_rt.timeline import Timeline  # noqa: E402
from hetero_rt.workloads import md as rmd  # noqa: E402

assert rk.NUMBA_ENABLED, "goldens pin the numba kernels (the reference default)"

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    "wall": rmd.MDParams(),  # the reference defaults: 10x10x24, 12 steps
    "per": rmd.MDParams(periodic=True, steps=10, dt=0.1),
    "tiny": rmd.MDParams(rows=2, cols=3, particles_per_patch=5, periodic=True, steps=9, dt=0.2, seed=3),
    "strip": rmd.MDParams(rows=1, cols=5, particles_per_patch=7, periodic=True, steps=6, seed=11),
    "sparse": rmd.MDParams(rows=7, cols=6, particles_per_patch=2, steps=15, dt=0.3, seed=19),
}


def run_case(p):
    wl = rmd.MDWorkload(p)
    tasks, inputs = [], []
    orig = wl._begin_step

    def begin(tl, start):
        work = rmd.pair_work(wl.grid, p.periodic)
        tasks.append(len(work))
        inputs.append(sum(1 if a == b else 2 for a, b, _ in work))
        orig(tl, start)

    wl._begin_step = begin
    cfg = ExperimentConfig(workload="md", md=p)
    tl = Timeline(cfg.device(), cfg.kernel_specs(wl.kernel_classes()), cfg.cost, cfg.policy_params())
    wl.setup(tl)
    tl.run()
    inv = {}
    consumed = {}
    for r in tl.runtime.invocations:
        inv[r.entry_method] = inv.get(r.entry_method, 0) + 1
        consumed[r.entry_method] = consumed.get(r.entry_method, 0) + r.messages_consumed
    g = wl.grid
    return {
        "pos": g.positions, "vel": g.velocities, "patch": g.patch_of,
        "tasks": np.array(tasks, np.int64), "inputs": np.array(inputs, np.int64),
        "inv_interact": inv.get("interact", 0), "inv_work_done": inv.get("work_done", 0),
        "inv_barrier": inv.get("step_barrier", 0), "msg_interact": consumed.get("interact", 0),
        "steps_done": wl.step,
    }


def main():
    out = {}
    for tag, p in CASES.items():
        r = run_case(p)
        for k, v in r.items():
            out[f"{tag}_{k}"] = np.asarray(v)
        for k, v in dataclasses.asdict(p).items():
            out[f"{tag}_param_{k}"] = np.asarray(v)
        print(tag, "steps", r["steps_done"], "tasks", r["tasks"].tolist()[:4], "inv", r["inv_interact"],
              r["inv_work_done"], r["inv_barrier"])
    path = os.path.join(HERE, "mdloop.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

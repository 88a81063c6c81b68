"""Closed-loop MD on the device: ms/step and per-phase time (10x10x24 and the
reference's 67x67x24 analogue, 107,736 atoms)."""
import json
import sys

sys.path.insert(0, ".")
from paper_2008_05712_b200.md import MDParams, MDWorkload  # noqa: E402

for rows, steps in ((10, 12), (67, 51), (67, 201)):
    p = MDParams(rows=rows, cols=rows, steps=steps, dt=0.02)
    MDWorkload(p).run()  # warm (module load, occupancy query)
    wl = MDWorkload(p)
    r = wl.run()
    ph = wl.phases_ns()[1:-1].mean(axis=0) / 1e3
    print(json.dumps({"grid": f"{rows}x{rows}x24", "atoms": len(wl.grid.positions), "steps": steps,
                      "device_ms": r.device_ms, "ms_per_step": r.device_ms / steps,
                      "phase_us": [round(float(x), 2) for x in ph],
                      "work_requests_per_step": int(r.work_requests.mean())}))

"""configs[0] through the device batcher once per memory mode (ncu launch-list driver + host timing)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2008_05712_b200 import generators as gen  # noqa: E402
from paper_2008_05712_b200 import nbody  # noqa: E402
from paper_2008_05712_b200.executor import GpuForceExecutor  # noqa: E402
from paper_2008_05712_b200.memory import MemoryMode  # noqa: E402

ps = gen.fp32_exact(gen.gen_plummer(16384, 42))
tree = nbody.build_bucket_tree(ps, 8)
lists = nbody.build_interaction_lists(tree, 0.7, ps)
lists.csr()
for mode in sys.argv[1:] or ["redundant", "reuse", "reuse_sorted"]:
    cap = 1 << 30 if mode == "redundant" else 64 << 20
    for rep in range(2):
        t0 = time.perf_counter()
        ex = GpuForceExecutor(tree, lists, MemoryMode.parse(mode), capacity_bytes=cap, slot_bytes=256, eps=1e-4)
        t1 = time.perf_counter()
        r = ex.run()
        print(mode, rep, f"ctor {1e3 * (t1 - t0):.2f} ms  run wall {1e3 * r.wall_s:.2f} ms  device {r.device_ms:.3f} ms",
              [round(b.device_ms, 3) for b in r.batches], flush=True)

# host-time breakdown of one phase (reuse mode)
import numpy as np  # noqa: E402
from paper_2008_05712_b200.executor import DeviceBatcher  # noqa: E402
ex = GpuForceExecutor(tree, lists, MemoryMode.REUSE, capacity_bytes=64 << 20, slot_bytes=256, eps=1e-4)
bat = ex.batcher
nb = len(ex.ptr) - 1
own = np.arange(nb)
t = np.zeros(nb)
for rep in range(2):
    if rep:
        ex = GpuForceExecutor(tree, lists, MemoryMode.REUSE, capacity_bytes=64 << 20, slot_bytes=256, eps=1e-4)
        bat = ex.batcher
    t0 = time.perf_counter()
    bat.submit(own, t, ex.ptr, ex.ids, ex.kind)
    t1 = time.perf_counter()
    bat.flush(0.0)
    t2 = time.perf_counter()
    rows, tms = bat.log()
    t3 = time.perf_counter()
    print(f"breakdown: submit {1e3 * (t1 - t0):.2f} ms  flush {1e3 * (t2 - t1):.2f} ms  log/sync {1e3 * (t3 - t2):.2f} ms "
          f"batches {len(rows)} device {tms[:, 1].sum():.3f} ms", flush=True)

"""Golden BH force stream of the REFERENCE's trace feed (hr/workloads/trace.py
nbody_stream), for tests/test_trace_cpu.py.  Dev container only:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_trace_golden.py
"""
import os
import sys

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from hetero_rt.workloads import nbody as rnb  # noqa: E402
from hetero_rt.workloads import trace as rtr  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
params = rnb.NBodyParams(particles=1500, bucket_size=8, theta=0.6, clustering=0.6, seed=5, dim=3)
rtr.dump_trace(rtr.nbody_stream(params), os.path.join(HERE, "trace_nbody3d_1500.txt"))
print("wrote", os.path.join(HERE, "trace_nbody3d_1500.txt"))

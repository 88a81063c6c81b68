#!/bin/bash
mkdir -p gpurun_out
GC_BUILD_PROF=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/r2i.log 2>&1
timeout 1200 python -m pytest tests/test_bh_gpu.py tests/test_bh_dist_gpu.py tests/test_trace_gpu.py tests/test_batcher_gpu.py tests/test_executor_gpu.py tests/test_dm_gpu.py -x -q -m gpu >> gpurun_out/r2i.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_bh_gpu.py tests/test_bh_dist_gpu.py tests/test_trace_gpu.py tests/test_batcher_gpu.py -m gpu > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
GC_BUILD_PROF=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/r2k_e2e.log 2>&1
GC_BUILD_PROF=1 timeout 300 python tools/e2e_breakdown.py 4194304 > gpurun_out/r2k_e2e4m.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_md_gpu.py tests/test_md_dist_gpu.py tests/test_executor_gpu.py tests/test_mdloop_gpu.py -x -m gpu > gpurun_out/r2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests.log
timeout 600 python tools/time_md8m.py > gpurun_out/r2j_time.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_bench.log 2>&1

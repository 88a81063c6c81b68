#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_md_gpu.py tests/test_md_dist_gpu.py tests/test_mdloop_gpu.py tests/test_bh_dist_gpu.py -x -m gpu > gpurun_out/r2s.log 2>&1; echo "rc=$?" >> gpurun_out/r2s.log
timeout 600 python tools/time_md8m.py >> gpurun_out/r2s.log 2>&1

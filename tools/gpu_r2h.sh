#!/bin/bash
# bottom-up device tree build: BH parity tests + e2e breakdown + build launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bh_gpu.py tests/test_bh_dist_gpu.py tests/test_trace_gpu.py -x -q -m gpu > gpurun_out/r2h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_tests.log
timeout 300 python tools/e2e_breakdown.py > gpurun_out/r2h_e2e.log 2>&1
timeout 300 python tools/e2e_breakdown.py 16777216 > gpurun_out/r2h_e2e16m.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bb_ --csv --log-file gpurun_out/r2h_build_launches.csv python tools/e2e_breakdown.py > /dev/null 2>&1

#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_bh_gpu.py -m gpu -k "handle_reuse or overlap" > gpurun_out/r2q.log 2>&1; echo "rc=$?" >> gpurun_out/r2q.log

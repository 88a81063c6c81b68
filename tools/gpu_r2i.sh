#!/bin/bash
mkdir -p gpurun_out
for c in 1 0 1 0; do echo "== climb $c"; GC_BUILD_CLIMB=$c timeout 300 python tools/e2e_breakdown.py | tail -3; done > gpurun_out/r2i.log 2>&1
GC_BUILD_CLIMB=0 timeout 600 python -m pytest tests/test_bh_gpu.py -x -q -m gpu -k "device_build or golden or digest or dyadic" >> gpurun_out/r2i.log 2>&1

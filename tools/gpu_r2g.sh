#!/bin/bash
# overlap mode 2 (fused walk+force kernel): parity + A/B over the force-first warp split
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bh_gpu.py -x -q -m gpu -k "overlap" > gpurun_out/r2g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_tests.log
for ff in 1 2 3 4 6; do
  echo "== force_first $ff" >> gpurun_out/r2g_overlap1m.log
  GC_WF_FORCE_FIRST=$ff timeout 300 python tools/time_overlap.py >> gpurun_out/r2g_overlap1m.log 2>&1
done
for ff in 2 4; do
  echo "== force_first $ff" >> gpurun_out/r2g_overlap4m.log
  GC_WF_FORCE_FIRST=$ff timeout 300 python tools/time_overlap.py 4000000 >> gpurun_out/r2g_overlap4m.log 2>&1
done

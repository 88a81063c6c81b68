#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/r2l.log
for i in 1 2; do
for lib in libgcharm_base.so libgcharm.so; do echo "== $lib" >> gpurun_out/r2l.log; GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py >> gpurun_out/r2l.log 2>&1; done
done
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_bh_gpu.py tests/test_bh_dist_gpu.py -m gpu -x >> gpurun_out/r2l.log 2>&1; echo "rc=$?" >> gpurun_out/r2l.log

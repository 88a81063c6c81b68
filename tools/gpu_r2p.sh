#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/r2p.log
for i in 1 2; do
for lib in libgcharm.so libgcharm_sh1.so; do echo "== $lib" >> gpurun_out/r2p.log; GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py >> gpurun_out/r2p.log 2>&1; done
done
GCHARM_LIB=$PWD/paper_2008_05712_b200/libgcharm_sh1.so timeout 900 python -m pytest -q -p no:cacheprovider tests/test_bh_gpu.py -m gpu -x >> gpurun_out/r2p.log 2>&1; echo "rc=$?" >> gpurun_out/r2p.log

#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/r2l.log
for i in 1 2; do
for lib in libgcharm.so libgcharm_u1.so libgcharm_u3.so libgcharm_u4.so; do echo "== $lib" >> gpurun_out/r2l.log; GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py >> gpurun_out/r2l.log 2>&1; done
done

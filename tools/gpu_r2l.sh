#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/r2l.log
for i in 1 2; do
for lib in libgcharm.so libgcharm_fl2.so libgcharm_fl4.so; do echo "== $lib" >> gpurun_out/r2l.log; GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py >> gpurun_out/r2l.log 2>&1; done
done
for lib in libgcharm_fl2.so libgcharm_fl4.so; do GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 600 python -m pytest -q -p no:cacheprovider tests/test_bh_gpu.py -m gpu -k "potential_energy_parity or tiny_softening or smoke or config3 or plummer16m" >> gpurun_out/r2l.log 2>&1; echo "$lib rc=$?" >> gpurun_out/r2l.log; done

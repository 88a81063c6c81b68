#!/bin/bash
# BH walk / force vs N on one GPU (clustered, theta 0.7)
mkdir -p gpurun_out
: > gpurun_out/r2u.log
for n in 1000000 2000000 4000000 8000000; do timeout 600 python tools/time_bh.py $n >> gpurun_out/r2u.log 2>&1; done

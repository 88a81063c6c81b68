#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/prof_dist.log
for i in 1 2; do timeout 900 python tools/prof_dist.py 2000000 2>&1 | head -1 >> gpurun_out/prof_dist.log; done

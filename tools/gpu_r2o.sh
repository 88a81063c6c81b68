#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/prof_dist.py 2000000 > gpurun_out/prof_dist.log 2>&1

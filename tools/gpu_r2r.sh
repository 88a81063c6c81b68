#!/bin/bash
# ncu --set full of the device tree build kernels (1M clustered, gc_bh_step path)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bb_" -s 20 -c 12 -o gpurun_out/prof_build python tools/e2e_breakdown.py > gpurun_out/ncu_build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bb_|Radix|Scan|Reduce" --csv --log-file gpurun_out/build_launches.csv python tools/e2e_breakdown.py > /dev/null 2>&1

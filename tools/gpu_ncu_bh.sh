cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"force_group|walk_group" -s 2 -c 2 -o gpurun_out/prof_bh python tools/prof_bh.py > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log

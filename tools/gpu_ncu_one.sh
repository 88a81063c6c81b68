# usage: gpu_ncu_one.sh <kernel regex> <out name>
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s 1 -c 1 -o gpurun_out/$2 python tools/prof_bh.py > gpurun_out/ncu_$2.log 2>&1
echo done >> gpurun_out/ncu_$2.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(timeout 300 python tools/time_bh.py; GCHARM_FG_NATURAL=1 timeout 300 python tools/time_bh.py) > gpurun_out/ab.log 2>&1

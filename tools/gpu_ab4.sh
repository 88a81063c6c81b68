cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/ab4.log
python -m pytest tests/test_bh_gpu.py tests/test_executor_gpu.py -x -q >> gpurun_out/ab4.log 2>&1
for rep in 1 2; do for lib in libgcharm.so "$@"; do GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py; done; done >> gpurun_out/ab4.log 2>&1

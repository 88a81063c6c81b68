cd $GRAFT_REPO_ROOT
: > gpurun_out/ab.log
python -m pytest tests/test_bh_gpu.py tests/test_sharding.py tests/test_executor_gpu.py tests/test_ewald_gpu.py -x -q >> gpurun_out/ab.log 2>&1
for rep in 1 2; do for lib in "$@"; do GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py; GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py staged; done; done >> gpurun_out/ab.log 2>&1
python tools/e2e_breakdown.py >> gpurun_out/ab.log 2>&1

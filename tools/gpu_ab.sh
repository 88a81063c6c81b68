cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "$@"; do GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py; done
done > gpurun_out/ab.log 2>&1
timeout 600 python -m pytest tests/test_bh_gpu.py -q -x -p no:cacheprovider >> gpurun_out/ab.log 2>&1
for lib in "$@"; do GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 600 python -m pytest tests/test_bh_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1; done >> gpurun_out/ab.log

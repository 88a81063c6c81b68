cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_md_gpu.py tests/test_md_dist_gpu.py tests/test_mdloop_gpu.py -x -q > gpurun_out/md_quick.log 2>&1
timeout 600 python tools/time_md8m.py >> gpurun_out/md_quick.log 2>&1

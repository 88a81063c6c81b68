cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_md_dist_gpu.py tests/test_batcher_gpu.py tests/test_executor_gpu.py -x > gpurun_out/r2e_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2e_tests.log
timeout 300 python tools/prof_batcher.py > gpurun_out/prof_batcher.log 2>&1

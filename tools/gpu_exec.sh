cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_executor_gpu.py tests/test_dm_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_exec.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_exec.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bh_gpu.py tests/test_sharding.py -q -p no:cacheprovider -x > gpurun_out/pytest_bh.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_bh.log
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e.log 2>&1
timeout 300 python tools/time_bh.py > gpurun_out/ab.log 2>&1

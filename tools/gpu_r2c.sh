cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_batcher_gpu.py tests/test_executor_gpu.py tests/test_dm_gpu.py -x > gpurun_out/batcher_tests.log 2>&1
echo "rc=$?" >> gpurun_out/batcher_tests.log
bash tools/gpu_md_col.sh
timeout 600 python -c "
import sys, time; sys.path.insert(0,'.')
import bench
class A: steps=3
print(bench.bench_runtime_path(A()))
" > gpurun_out/runtime_path.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_trace_gpu.py tests/test_executor_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_misc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_misc.log
GCHARM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench4.log 2>&1
echo "rc=$?" >> gpurun_out/bench4.log

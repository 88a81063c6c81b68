# N > 1 dry run of bench.py on one GPU: 2 gloo ranks sharing cuda:0
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
GCHARM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/dist_bench.log 2>&1
echo "rc=$?" >> gpurun_out/dist_bench.log

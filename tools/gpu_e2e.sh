cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e.log 2>&1
timeout 300 nsys --version >> gpurun_out/e2e.log 2>&1

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/prof_batcher.py > gpurun_out/prof_batcher.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/batcher_launches.csv python tools/prof_batcher.py reuse > /dev/null 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_trace_gpu.py > gpurun_out/trace_tests.log 2>&1
echo "rc=$?" >> gpurun_out/trace_tests.log

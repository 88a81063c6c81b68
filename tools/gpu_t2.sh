python -m pytest tests/test_bh_gpu.py tests/test_sharding.py -x -q > gpurun_out/t2.log 2>&1; echo "rc=$?" >> gpurun_out/t2.log
python tools/e2e_breakdown.py >> gpurun_out/t2.log 2>&1

timeout 300 python -m pytest tests/test_bh_gpu.py -x -q > gpurun_out/t4.log 2>&1
timeout 200 python tools/time_overlap.py >> gpurun_out/t4.log 2>&1
timeout 200 python tools/time_bh.py >> gpurun_out/t4.log 2>&1

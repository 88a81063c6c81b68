python -m pytest tests/test_mdloop_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/mdloop_test.log
python tools/time_mdloop.py > gpurun_out/mdloop_time.log 2>&1
echo done

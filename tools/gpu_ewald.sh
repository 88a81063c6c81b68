python -m pytest tests/test_ewald_gpu.py tests/test_executor_gpu.py tests/test_mdloop_gpu.py -x -q 2>&1 | tail -25 > gpurun_out/ewald_test.log
python tools/time_mdloop.py > gpurun_out/mdloop_time.log 2>&1
GCHARM_LIB=build/ab/libgcharm_b.so python tools/time_mdloop.py > gpurun_out/mdloop_time_b.log 2>&1
echo done

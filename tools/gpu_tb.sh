python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/time_mdloop.py > gpurun_out/mdloop_time.log 2>&1
GCHARM_LIB=$PWD/paper_2008_05712_b200/libgcharm_ml1.so python tools/time_mdloop.py > gpurun_out/mdloop_time_ml1.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
echo done

python -m pytest tests -m gpu -x -q > gpurun_out/t2.log 2>&1; echo "rc=$?" >> gpurun_out/t2.log
python tools/e2e_breakdown.py >> gpurun_out/t2.log 2>&1
python tools/time_bh.py >> gpurun_out/t2.log 2>&1

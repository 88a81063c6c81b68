timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e2e_launches.csv python tools/e2e_breakdown.py > gpurun_out/e2e_ncu.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_md_gpu.py tests/test_md_dist_gpu.py tests/test_executor_gpu.py -x -m gpu > gpurun_out/r2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests.log
timeout 600 python tools/time_md8m.py > gpurun_out/r2j_time.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_md8m_launches.csv python -c "import sys; sys.path.insert(0,\".\"); from paper_2008_05712_b200 import md; from paper_2008_05712_b200.generators import gen_lj_fcc; s=md.LJSystem(gen_lj_fcc(126)); s.run(2)" > /dev/null 2>&1 || true

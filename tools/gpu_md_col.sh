# MD column kernel: GPU tests, configs[4] timing, ncu of the LJ cell kernel at 8M
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_md_gpu.py tests/test_md_dist_gpu.py -x > gpurun_out/mdcol_tests.log 2>&1
echo "rc=$?" >> gpurun_out/mdcol_tests.log
timeout 600 python tools/time_md8m.py > gpurun_out/mdcol_time.log 2>&1
cat > /tmp/md8m_one.py <<'PY'
import sys
sys.path.insert(0, '.')
from paper_2008_05712_b200 import md
from paper_2008_05712_b200.generators import gen_lj_fcc
s = gen_lj_fcc(126)
sysd = md.LJSystem(s)
sysd.run(2)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/md8m_launches.csv python /tmp/md8m_one.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"md_lj3" -s 1 -c 1 -o gpurun_out/prof_md8m_col python /tmp/md8m_one.py > gpurun_out/ncu_md8m_col.log 2>&1

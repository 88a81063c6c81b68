cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_md_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_md.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_md.log
timeout 600 python - > gpurun_out/md_timing.log 2>&1 <<'PY'
import sys, time
sys.path.insert(0, '.')
from paper_2008_05712_b200 import md
from paper_2008_05712_b200.generators import gen_lj_fcc
s = gen_lj_fcc(30)
sysd = md.LJSystem(s)
sysd.run(100)
for _ in range(3):
    print("100 steps ms", sysd.run(100))
f, e = sysd.forces()
print("force-only ms", sysd.dev.elapsed_ms())
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/md_launches.csv python -c "
import sys; sys.path.insert(0, '.')
from paper_2008_05712_b200 import md
from paper_2008_05712_b200.generators import gen_lj_fcc
s = md.LJSystem(gen_lj_fcc(30)); s.run(3)" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_md_dist_gpu.py tests/test_md_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_md.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_md.log

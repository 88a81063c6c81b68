# Round-2 measurement pass: full GPU tests + smoke, bench (N=1), launch list of the bench,
# ncu --set full of the BH kernels at 1M and 16M and of the LJ kernel at 8M.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"force_fused|walk_group|expand|force_group" -s 2 -c 5 -o gpurun_out/prof_bh1m python tools/prof_bh.py > gpurun_out/ncu_bh1m.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"force_fused|walk_group" -s 2 -c 2 -o gpurun_out/prof_bh16m python tools/prof_bh16m.py > gpurun_out/ncu_bh16m.log 2>&1
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
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"md_lj3c|md_sortgather|md_integrate" -s 3 -c 3 -o gpurun_out/prof_md8m python /tmp/md8m_one.py > gpurun_out/ncu_md8m.log 2>&1

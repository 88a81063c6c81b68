# ncu --set full of force_fused_kernel (1M clustered) for the current library and the variants named
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in libgcharm.so "$@"; do
  tag=${lib%.so}
  GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"force_fused" -s 1 -c 1 -o gpurun_out/prof_$tag python tools/prof_bh.py > gpurun_out/ncu_$tag.log 2>&1
done
# MD configs[4] system: the LJ cell kernel at 8M
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
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"md_lj3" -s 1 -c 1 -o gpurun_out/prof_md8m python /tmp/md8m_one.py > gpurun_out/ncu_md8m.log 2>&1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/mdprof.py <<'PY'
import sys
sys.path.insert(0, '.')
from paper_2008_05712_b200 import md
from paper_2008_05712_b200.generators import gen_lj_fcc
s = gen_lj_fcc(30)
sysd = md.LJSystem(s)
sysd.forces(); sysd.forces()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"md_cell_kernel" -s 1 -c 1 -o gpurun_out/prof_md python /tmp/mdprof.py > gpurun_out/ncu_md.log 2>&1

# A/B of LJ 8M force time for the current library and the variants named
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/md_ab.log
for lib in libgcharm.so "$@"; do echo "== $lib" >> gpurun_out/md_ab.log; GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_md8m.py >> gpurun_out/md_ab.log 2>&1; done
GCHARM_LIB=$PWD/paper_2008_05712_b200/${1:-libgcharm.so} timeout 600 python -m pytest -q -p no:cacheprovider tests/test_md_gpu.py tests/test_md_dist_gpu.py -x >> gpurun_out/md_ab.log 2>&1

# A/B: bit-identity + parity tests of the current library, then times of the
# current library vs the variants named on the command line (1M clustered)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/ab5.log
timeout 900 python -m pytest tests/test_bh_gpu.py -x -q -p no:cacheprovider >> gpurun_out/ab5.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab5.log
for rep in 1 2; do for lib in libgcharm.so "$@"; do GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 300 python tools/time_bh.py; done; done >> gpurun_out/ab5.log 2>&1

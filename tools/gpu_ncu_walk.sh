# ncu --set full of walk_group_kernel (1M clustered) for the current library and the variants named
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in libgcharm.so "$@"; do
  tag=${lib%.so}
  GCHARM_LIB=$PWD/paper_2008_05712_b200/$lib timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"walk_group" -s 1 -c 1 -o gpurun_out/profw_$tag python tools/prof_bh.py > gpurun_out/ncuw_$tag.log 2>&1
done

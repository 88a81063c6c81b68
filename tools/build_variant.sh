#!/bin/bash
# build_variant.sh NAME "NVCC FLAGS": an A/B copy of libgcharm.so with extra
# defines -> paper_2008_05712_b200/libgcharm_NAME.so (git-ignored; travels with gpurun)
set -e
name=$1; shift
flags="$*"
# SRC=<dir> builds the sources of another tree (e.g. a `git archive` of an older commit)
root="$(cd "$(dirname "$0")/.." && pwd)"
cd "${SRC:-$root/paper_2008_05712_b200/csrc}"
out=$root/build/var_$name
mkdir -p $out
objs=""
for f in abi.cu bh.cu bh_build.cu md.cu md_loop.cu ewald.cu dm.cu $( [ -f batcher.cu ] && echo batcher.cu ); do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
       --expt-relaxed-constexpr $flags -c $f -o $out/$f.o &
  objs="$objs $out/$f.o"
done
wait
if [ -f bh_tree.cpp ]; then  # older trees still had the host builder
  nvcc -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -c bh_tree.cpp -o $out/bh_tree.o
  objs="$objs $out/bh_tree.o"
fi
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $root/paper_2008_05712_b200/libgcharm_$name.so $objs -lcudart
echo built libgcharm_$name.so

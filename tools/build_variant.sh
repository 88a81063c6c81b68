#!/bin/bash
# build_variant.sh NAME "NVCC FLAGS": an A/B copy of libgcharm.so with extra
# defines -> paper_2008_05712_b200/libgcharm_NAME.so (git-ignored; travels with gpurun)
set -e
name=$1; shift
flags="$*"
cd "$(dirname "$0")/../paper_2008_05712_b200/csrc"
out=../../build/var_$name
mkdir -p $out
objs=""
for f in abi.cu bh.cu bh_build.cu md.cu md_loop.cu ewald.cu dm.cu; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
       --expt-relaxed-constexpr $flags -c $f -o $out/$f.o &
  objs="$objs $out/$f.o"
done
wait
nvcc -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -c bh_tree.cpp -o $out/bh_tree.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libgcharm_$name.so $objs $out/bh_tree.o -lcudart
echo built ../libgcharm_$name.so

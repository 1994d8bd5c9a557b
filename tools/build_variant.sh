#!/bin/bash
# Build an experimental libb200hot.so with extra nvcc defines into exp_builds/<tag>/
# usage: tools/build_variant.sh <tag> -DFOO=1 ...
tag=$1; shift
out=exp_builds/$tag
mkdir -p $out
P=paper_2504_19516_b200
objs=""
for f in $P/csrc/*.cu; do
  o=$out/$(basename $f .cu).o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude -I$P/csrc "$@" -c $f -o $o &
  objs="$objs $o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libb200hot.so $objs
echo $out/libb200hot.so

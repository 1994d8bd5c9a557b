#!/bin/bash
# experiment builds: $1 = output dir, rest = extra nvcc flags
set -e
D=$1; shift; rm -rf $D; mkdir -p $D
cd /root/repo/paper_2504_19516_b200/csrc
for f in *.cu; do /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -I/root/repo/include -I. -c $f -o $D/${f%.cu}.o 2>/dev/null & done; wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $D/libb200hot.so $D/*.o

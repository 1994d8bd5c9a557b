#!/bin/bash
# compute-sanitizer memcheck over every hot-path kernel (small shapes).
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for k in "gemm1024 148 1" "swap 148 1" "swap_qkv 32 1" "decode_attn 148 1" "decode_attn 8 1" "attn1024 148 1"; do
  set -- $k
  timeout 600 $CS --tool memcheck --print-limit 20 python tools/one_kernel.py $1 $2 $3 > $OUT/memcheck_$1_$2.txt 2>&1
  echo "$1 $2: $(grep -c 'Invalid\|ERROR SUMMARY' $OUT/memcheck_$1_$2.txt) $(grep 'ERROR SUMMARY' $OUT/memcheck_$1_$2.txt)"
done
timeout 900 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_kernels_gpu.py -q -x -k "paged or qkv_rope or decode_attn" > $OUT/memcheck_pytest.txt 2>&1
echo "pytest: $(grep 'ERROR SUMMARY\|passed\|failed' $OUT/memcheck_pytest.txt | tail -3)"

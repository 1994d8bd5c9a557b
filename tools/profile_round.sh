#!/bin/bash
# Round profile capture (run under gpurun): bench line, ncu launch list of the
# same bench command, and one full ncu capture of each dominant kernel.
# Usage: bash tools/profile_round.sh <tag> [pm_sms] [split pm,dm]
TAG=${1:-r01}
PM=${2:-140}
SPLIT=${3:-}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | head -20 >> $OUT/nproc.txt
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
tail -c 3000 $OUT/bench.err
cat $OUT/bench.json
if [ -z "$SPLIT" ]; then
  SPLIT=$(python -c "import json;d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]);c=d['split'];print(f\"{c['pm']},{c['dm']}\")")
fi
echo "split $SPLIT"
# launch list of the same bench command (fixed split, no sweep): every launch.
# HP_NO_GREEN=1: plain streams with the split's grid sizes (ncu cannot prepare
# kernels launched into green-context streams on this driver)
HP_NO_GREEN=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sweep "" \
    --no-regret-sweep --split $SPLIT > $OUT/ncu_bench.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 6 -c 1 \
    -o $OUT/upgate python tools/one_kernel.py gemm4096 $PM 8 > $OUT/ncu_upgate.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 2 -c 1 \
    -o $OUT/decode_attn python tools/one_kernel.py decode_attn 148 4 > $OUT/ncu_dattn.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fa2 -s 1 -c 1 \
    -o $OUT/prefill_attn python tools/one_kernel.py attn4096 $PM 3 > $OUT/ncu_fa.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_swap -s 2 -c 1 \
    -o $OUT/swap_o python tools/one_kernel.py swap 148 4 > $OUT/ncu_swap.out 2>&1
# the decode partition's view: CTA-pair decode GEMM (mlp_up_gate) and decode attention on 8 SMs
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_swap -s 2 -c 1 \
    -o $OUT/swap_ug8 python tools/one_kernel.py swap_ug 8 4 > $OUT/ncu_swap8.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 2 -c 1 \
    -o $OUT/decode_attn8 python tools/one_kernel.py decode_attn 8 4 > $OUT/ncu_dattn8.out 2>&1
# the dual-roofline split's decode side (dm = 88 >= n_d)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 2 -c 1 \
    -o $OUT/decode_attn88 python tools/one_kernel.py decode_attn 88 4 > $OUT/ncu_dattn88.out 2>&1
ls -la $OUT

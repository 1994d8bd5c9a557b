#!/bin/bash
# Config-4 real-time serving sweep on one B200 (run under gpurun).
# usage: tools/serve_sweep.sh OUTDIR "RATE:POLICIES:SLO_MS ..."
out=$1; shift
mkdir -p "$out"
for spec in $1; do
  IFS=: read rate pols slo <<< "$spec"
  tag="r${rate}_${pols//,/-}_${slo//,/-}"
  python -m paper_2504_19516_b200.device.serve --rate "$rate" --duration 10 --policies "$pols" \
      ${slo:+--slo-ms $slo} --out "$out/$tag.jsonl" > "$out/$tag.log" 2>&1 || echo "FAILED $tag"
done

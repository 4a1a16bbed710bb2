#!/bin/bash
# A/B of kernel choices at the per-rank batch of 2/4/8-GPU cfg5 runs
cd "$(dirname "$0")/.."
for B in 2048 4096 8192; do
  for m in "" "SP_SPMM_SK=1" "SP_SPMM_SK=0" "SP_FUSED_HALF=0"; do
    echo "== B=$B $m" >> gpurun_out/ab_smallb.log
    (env $m timeout 120 python tools/prof_layer.py --B $B; env $m timeout 120 python tools/prof_layer.py --B $B --R 768 --C 3072) 2>&1 | grep -E "fwd|fused" | tr '\n' ' ' >> gpurun_out/ab_smallb.log
    echo >> gpurun_out/ab_smallb.log
  done
done

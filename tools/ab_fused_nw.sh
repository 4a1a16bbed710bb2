#!/bin/bash
# fused backward: warps-per-CTA variants (half-warp entries) on the cfg5 layer shapes
cd "$(dirname "$0")/.."
for m in "" "SP_FUSED_NW=28" "SP_FUSED_NW=24" "SP_FUSED_NW=16"; do
  echo "== $m" >> gpurun_out/ab_fused_nw.log
  (env $m timeout 120 python tools/prof_layer.py; env $m timeout 120 python tools/prof_layer.py --R 768 --C 3072) 2>&1 | grep -E "fused" | tr '\n' ' ' >> gpurun_out/ab_fused_nw.log
  echo >> gpurun_out/ab_fused_nw.log
done

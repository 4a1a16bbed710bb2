#!/bin/bash
# gather kernels vs staged tiles on the small-batch configs (cfg2 B=512, cfg1, B=2048 layers)
cd "$(dirname "$0")/.."
for m in "" "SP_GATHER=1"; do
  echo "== $m" >> gpurun_out/ab_gather.log
  (env $m timeout 120 python tools/prof_layer.py --B 512; env $m timeout 120 python tools/prof_layer.py --B 512 --R 768 --C 3072; env $m timeout 120 python tools/prof_layer.py --B 2048) 2>&1 | tr '\n' ' ' >> gpurun_out/ab_gather.log
  echo >> gpurun_out/ab_gather.log
done

#!/bin/bash
# ncu --set full (with source) of the cfg5-shape fused backward and forward kernels
cd "$(dirname "$0")/.."
T=${1:-g0}
python tools/prof_layer.py --iters 1 > gpurun_out/${T}_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:bwd_fused' -s 0 -c 2 \
   -o gpurun_out/${T}_full python tools/prof_layer.py --iters 1 > gpurun_out/${T}_full.log 2>&1
echo done > gpurun_out/${T}_done

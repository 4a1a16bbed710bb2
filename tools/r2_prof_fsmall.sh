#!/bin/bash
# ncu --set full of the fused backward at the small-batch shapes (cfg2a, cfg4 95%)
cd "$(dirname "$0")/.."
T=${1:-f0}
python tools/prof_layer.py --B 512 --iters 1 > gpurun_out/${T}_plain.log 2>&1 || exit 1
python tools/prof_cfg4.py --sparsity 0.95 --kind uniform --iters 1 >> gpurun_out/${T}_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_fused -s 1 -c 1 \
   -o gpurun_out/${T}_b512 python tools/prof_layer.py --B 512 --iters 1 > gpurun_out/${T}_b512.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_fused -s 1 -c 1 \
   -o gpurun_out/${T}_c4 python tools/prof_cfg4.py --sparsity 0.95 --kind uniform --iters 1 > gpurun_out/${T}_c4.log 2>&1
echo done > gpurun_out/${T}_done

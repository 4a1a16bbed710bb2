#!/bin/bash
# ncu evidence for the single-layer configs (round 2): per-launch durations and
# --set full of the hot kernels for cfg4 95% / 99% uniform and cfg2a.
cd "$(dirname "$0")/.."
T=${1:-s0}
K='regex:spmm|fused|sddmm|gather|job_reduce|refresh|reduce'
python tools/prof_cfg4.py --sparsity 0.95 --kind uniform --iters 2 > gpurun_out/${T}_plain.log 2>&1 || exit 1
python tools/prof_cfg4.py --sparsity 0.99 --kind uniform --iters 2 >> gpurun_out/${T}_plain.log 2>&1 || exit 1
python tools/prof_layer.py --B 512 --iters 2 >> gpurun_out/${T}_plain.log 2>&1 || exit 1
for a in "cfg4 --sparsity 0.95 --kind uniform" "cfg4 --sparsity 0.99 --kind uniform" "layer --B 512"; do
  set -- $a; n=$1; shift
  if [ $n = cfg4 ]; then s=tools/prof_cfg4.py; else s=tools/prof_layer.py; fi
  tag=$(echo "$n$*" | tr -d ' -.')
  timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread --clock-control none -k "$K" --csv \
     python $s "$@" --iters 2 > gpurun_out/${T}_launch_$tag.csv 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k "$K" -s 0 -c 8 \
     -o gpurun_out/${T}_full_$tag python $s "$@" --iters 1 > gpurun_out/${T}_full_$tag.log 2>&1
done
echo done > gpurun_out/${T}_done

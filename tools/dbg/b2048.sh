#!/bin/bash
# kernel durations of the cfg5 layer shapes at the per-rank batch of an 8-GPU run (B = 2048)
cd "$(dirname "$0")/../.."
for rc in "3072 768" "768 3072"; do
  set -- $rc
  python tools/prof_layer.py --B 2048 --R $1 --C $2 --iters 2 > gpurun_out/b2048_plain_$1.log 2>&1 &&
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b2048_$1.csv \
      python tools/prof_layer.py --B 2048 --R $1 --C $2 --iters 2 > gpurun_out/b2048_ncu_$1.log 2>&1
done

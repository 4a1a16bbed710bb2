#!/bin/bash
# per-kernel durations at the per-rank batch of a 4- and 8-GPU cfg5 run
cd "$(dirname "$0")/.."
for B in 2048 4096; do
for RC in "3072 768" "768 3072"; do
  set -- $RC
  timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
    python tools/prof_layer.py --B $B --R $1 --C $2 --iters 2 > gpurun_out/sb_${B}_$1.csv 2>&1
  timeout 120 python tools/prof_layer.py --B $B --R $1 --C $2 >> gpurun_out/sb_events.log 2>&1
done; done

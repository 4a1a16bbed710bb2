#!/bin/bash
# per-kernel durations (ncu launch list) of the small-batch / very sparse configs
cd "$(dirname "$0")/.."
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
  python tools/prof_layer.py --B 512 --iters 2 > gpurun_out/small_cfg2.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
  python tools/prof_cfg4.py --sparsity 0.99 --kind zipf --iters 2 > gpurun_out/small_z99.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv \
  python tools/prof_cfg4.py --sparsity 0.99 --kind uniform --iters 2 > gpurun_out/small_u99.csv 2>&1

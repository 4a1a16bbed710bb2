#!/bin/bash
# A/B: conv tap-tile skip and split rows (variants noskip / nosplit vs default), 3 rounds interleaved
cd "$(dirname "$0")/.."
T=$1
for rep in 1 2 3; do
for v in default noskip nosplit; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v conv" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L python tools/prof_conv.py --iters 10 >> gpurun_out/${T}_ab.log 2>&1
  for s in 0.8 0.95 0.99; do
    echo "== $v zipf$s" >> gpurun_out/${T}_ab.log
    SPARSEPROP_LIB=$L python tools/prof_cfg4.py --sparsity $s --kind zipf --iters 10 >> gpurun_out/${T}_ab.log 2>&1
  done
done; done

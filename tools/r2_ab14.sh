#!/bin/bash
# A/B on the cfg5 layer shapes at B = 16384 / 2048 and the staged single-layer configs
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg5w1 cfg5w2 cfg2a@2048 cfg2b@2048 cfg2a cfg2b cfg4:uniform:0.95 cfg3 >> gpurun_out/${T}_ab.log 2>&1
done

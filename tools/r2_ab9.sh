#!/bin/bash
# A/B of variant libraries on the cfg5 layer shapes and the staged single-layer configs
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg5w1 cfg5w2 cfg2a cfg2b cfg4:uniform:0.95 cfg4:uniform:0.9 cfg3 >> gpurun_out/${T}_ab.log 2>&1
done

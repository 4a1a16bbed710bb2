#!/bin/bash
# A/B on the small-batch layer shapes (cfg2a / cfg2b and the cfg5 shapes at B = 1024 / 2048)
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg2a cfg2b cfg2a@1024 cfg2b@1024 cfg2a@2048 cfg2b@2048 >> gpurun_out/${T}_ab.log 2>&1
done

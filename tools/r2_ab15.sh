#!/bin/bash
# A/B on the 768-row (cfg2b / cfg5 W2) forward at B = 512 .. 4096
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg2b cfg2b@1024 cfg2b@2048 cfg2b@4096 cfg2a@2048 cfg2a@4096 >> gpurun_out/${T}_ab.log 2>&1
done

#!/bin/bash
# A/B on the forward SpMMs (cfg5 shapes, cfg4 95 %, cfg2)
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg5w1 cfg5w2 cfg4:uniform:0.95 cfg4:uniform:0.9 cfg2a cfg2b >> gpurun_out/${T}_ab.log 2>&1
done

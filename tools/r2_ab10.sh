#!/bin/bash
# A/B of variant libraries on the configs the tiled SpMM serves (cfg4 80 / 90 %, cfg2 shapes, conv direct)
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg4:uniform:0.8 cfg4:uniform:0.9 cfg4:zipf:0.8 cfg4:zipf:0.9 cfg2a cfg5w1 >> gpurun_out/${T}_ab.log 2>&1
done

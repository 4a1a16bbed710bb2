#!/bin/bash
# A/B of variant libraries on the gather-regime configs (98-99 %, uniform and Zipf, B = 128 / 256 / 512)
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg4:uniform:0.99 cfg4:uniform:0.98 cfg4:zipf:0.99 cfg4:zipf:0.98 cfg4:uniform:0.99:512 cfg4:zipf:0.99:512 cfg4:uniform:0.99:128 >> gpurun_out/${T}_ab.log 2>&1
done

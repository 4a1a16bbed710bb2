#!/bin/bash
# A/B on cfg3 (conv) only
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 300 python tools/cfg_time.py cfg3 cfg3 >> gpurun_out/${T}_ab.log 2>&1
done

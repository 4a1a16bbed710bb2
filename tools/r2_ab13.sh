#!/bin/bash
# A/B on the configs whose kernels pair a producer with a reduction (Zipf split rows, fused + job reduce)
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg4:zipf:0.8 cfg4:zipf:0.9 cfg4:zipf:0.95 cfg4:zipf:0.99 cfg2a cfg2b cfg4:uniform:0.95 >> gpurun_out/${T}_ab.log 2>&1
done

#!/bin/bash
# A/B of single-layer configs between library builds (graph-replayed, L2-flushed:
# tools/cfg_time.py).  usage: tools/ab_cfgs.sh TAG "cfg list" variant...  (default = the product build)
cd "$(dirname "$0")/.."
T=$1; CF=$2; shift 2
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py $CF >> gpurun_out/${T}_ab.log 2>&1
done

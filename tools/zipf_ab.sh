#!/bin/bash
# cfg4 Zipf forward under the SpMM kernel choices
cd "$(dirname "$0")/.."
for s in 0.99 0.98 0.95; do
  for m in "" "SP_SPMM_SK=0" "SP_SPMM_SK=1"; do
    echo "== $s $m" >> gpurun_out/zipf_ab.log
    env $m timeout 120 python tools/prof_cfg4.py --sparsity $s >> gpurun_out/zipf_ab.log 2>&1
  done
done
timeout 120 python tools/prof_cfg4.py --sparsity 0.99 --kind uniform >> gpurun_out/zipf_ab.log 2>&1

#!/bin/bash
# TMEM-gather SpMM timing experiments (wrong results in dbg modes): full / no copies / no compute / neither
cd "$(dirname "$0")/.."
export SP_SPMM_TM=1
for v in ${VARS:-1}; do for d in ${DBGS:-0 1 2 3}; do
  echo "== variant $v dbg $d" >> gpurun_out/tm_dbg.log
  SP_SPMM_TM_VAR=$v SP_SPMM_TM_DBG=$d timeout 120 python tools/prof_layer.py 2>&1 | grep fwd >> gpurun_out/tm_dbg.log
done; done
SP_SPMM_TM_VAR=1 timeout 120 python tools/prof_layer.py --iters 1 > /dev/null 2>&1
SP_SPMM_TM_VAR=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmm_tm -c 1 -o gpurun_out/tm_full python tools/prof_layer.py --iters 1 > gpurun_out/tm_ncu.log 2>&1

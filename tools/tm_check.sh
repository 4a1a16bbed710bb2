#!/bin/bash
# TMEM-gather SpMM check under gpurun: parity tests with SP_SPMM_TM=1, then cfg5 layer timings per variant.
cd "$(dirname "$0")/.."
export SP_SPMM_TM=1
timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "${1:-cfg1 or cfg2 or cfg4 or ragged or relu or determinism or empty}" > gpurun_out/tm_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tm_tests.log
for v in 0 1; do
  echo "== variant $v" >> gpurun_out/tm_layer.log
  (SP_SPMM_TM_VAR=$v timeout 120 python tools/prof_layer.py; SP_SPMM_TM_VAR=$v timeout 120 python tools/prof_layer.py --R 768 --C 3072) >> gpurun_out/tm_layer.log 2>&1
done

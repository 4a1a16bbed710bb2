#!/bin/bash
# split-source SpMM: parity (subprocess test) + cfg5 layer timings with and without
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_ab_switches_gpu.py -x -q -k hyb > gpurun_out/hyb_tests.log 2>&1
echo "rc=$?" >> gpurun_out/hyb_tests.log
for m in 0 1; do
  echo "== SP_SPMM_HYB=$m" >> gpurun_out/hyb_layer.log
  (SP_SPMM_HYB=$m timeout 120 python tools/prof_layer.py; SP_SPMM_HYB=$m timeout 120 python tools/prof_layer.py --R 768 --C 3072) 2>&1 | grep -E "fwd|dx" >> gpurun_out/hyb_layer.log
done

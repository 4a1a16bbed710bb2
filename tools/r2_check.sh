#!/bin/bash
# GPU check: selected (or all) gpu tests, then bench.py (with the per-config sweep)
cd "$(dirname "$0")/.."
T=${1:-c0}; K=${2:-}
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${T}_tests.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1
fi
echo "tests rc=$?" >> gpurun_out/${T}_tests.log
timeout 600 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${T}_bench.log

#!/bin/bash
# quick GPU check used during kernel work: parity tests matching $1 + cfg5 layer timings
cd "$(dirname "$0")/.."
python -m pytest tests/test_parity_gpu.py -x -q -k "${1:-fused}" > gpurun_out/q_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/q_tests.log
(python tools/prof_layer.py; python tools/prof_layer.py --R 768 --C 3072) > gpurun_out/q_layer.log 2>&1

#!/bin/bash
# A/B layer timings: $1 = env assignment for the B arm (e.g. SP_SPMM_SK=0); shapes: cfg5 x2, cfg2, cfg4@90
cd "$(dirname "$0")/.."
for args in "" "--R 768 --C 3072" "--B 512" "--R 4096 --C 4096 --B 256 --density 0.1" "--R 4096 --C 4096 --B 256 --density 0.2"; do
  echo "== $args"
  python tools/prof_layer.py $args | sed 's/^/A_/'
  env $1 python tools/prof_layer.py $args | sed 's/^/B_/'
done

#!/bin/bash
cd "$(dirname "$0")/../.."
for v in "$@"; do
  L=""; [ "$v" != default ] && L=paper_2302_04852_b200/build/variants/$v.so
  SPARSEPROP_LIB=$L python tools/prof_conv.py --iters 2 > /dev/null 2>&1
  SPARSEPROP_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/jr_$v.csv python tools/prof_conv.py --iters 2 > /dev/null 2>&1
  SPARSEPROP_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/jr5_$v.csv python tools/prof_layer.py --iters 2 > /dev/null 2>&1
done

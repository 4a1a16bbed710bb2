#!/bin/bash
# run the bench launch-list command under ncu with each library variant
cd "$(dirname "$0")/../.."
for v in "$@"; do
  L=paper_2302_04852_b200/build/variants/$v.so
  SPARSEPROP_LIB=$L timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bis_$v.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/bis_$v.log 2>&1
  echo "$v rc=$? $(grep -c '' gpurun_out/bis_$v.csv) $(grep -c LaunchFailed gpurun_out/bis_$v.csv)" >> gpurun_out/bis_summary.txt
done

#!/bin/bash
# A/B of variants on small-batch shapes: tools/r2_ab2.sh TAG variant...
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  for rep in 1 2; do
  for args in "--R 3072 --C 768 --B 512" "--R 768 --C 3072 --B 512" "--R 4096 --C 4096 --B 256" "--R 4096 --C 4096 --B 256 --density 0.02" "--R 3072 --C 768 --B 1024" "--R 256 --C 256 --B 32 --density 0.1"; do
    echo "== $v $args" >> gpurun_out/${T}_ab.log
    SPARSEPROP_LIB=$L timeout 120 python tools/prof_layer.py --iters 15 $args >> gpurun_out/${T}_ab.log 2>&1
  done; done
done
echo done >> gpurun_out/${T}_ab.log

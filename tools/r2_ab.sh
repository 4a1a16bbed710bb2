#!/bin/bash
# A/B of library variants (build/variants/*.so) on the cfg5 layer shapes and cfg4/cfg2:
# usage: r2_ab.sh TAG variant1 variant2 ...   ("default" = the product build)
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  for rep in 1 2; do
  for args in "--R 3072 --C 768" "--R 768 --C 3072" "--R 3072 --C 768 --B 2048" "--R 4096 --C 4096 --B 256" "--R 3072 --C 768 --B 512"; do
    echo "== $v $args" >> gpurun_out/${T}_ab.log
    SPARSEPROP_LIB=$L timeout 120 python tools/prof_layer.py --iters 15 $args >> gpurun_out/${T}_ab.log 2>&1
  done; done
done
echo done >> gpurun_out/${T}_ab.log

#!/bin/bash
# A/B: gather SpMM entries in flight (default 8 vs variant gu4)
cd "$(dirname "$0")/.."
T=$1
for rep in 1 2; do
for v in default gu4; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  for a in "0.99 uniform" "0.98 uniform" "0.99 zipf"; do set -- $a
    echo "== $v $1 $2" >> gpurun_out/${T}_ab.log
    SPARSEPROP_LIB=$L python tools/prof_cfg4.py --sparsity $1 --kind $2 --iters 10 >> gpurun_out/${T}_ab.log 2>&1
  done
  echo "== $v cfg1" >> gpurun_out/${T}_ab.log
  SPARSEPROP_LIB=$L python tools/prof_layer.py --R 256 --C 256 --B 32 --density 0.1 --iters 10 >> gpurun_out/${T}_ab.log 2>&1
done; done
python tools/create_time.py > gpurun_out/${T}_create.log 2>&1

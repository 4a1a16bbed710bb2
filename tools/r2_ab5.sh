#!/bin/bash
cd "$(dirname "$0")/.."
T=$1
for rep in 1 2; do
for v in default gu16; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  for a in "0.99 uniform" "0.98 uniform"; do set -- $a
    echo "== $v $1 $2" >> gpurun_out/${T}_ab.log
    SPARSEPROP_LIB=$L python tools/prof_cfg4.py --sparsity $1 --kind $2 --iters 10 >> gpurun_out/${T}_ab.log 2>&1
  done
done; done
python tools/create_time.py > gpurun_out/${T}_create.log 2>&1
python -m pytest tests -m gpu -x -q -k "big_handle or nn_gpu or create or cfg1 or empty or ragged" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log

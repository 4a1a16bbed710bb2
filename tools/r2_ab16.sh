#!/bin/bash
# A/B of variant libraries on the whole DP step (16384 and 2048 tokens) and the single-layer configs
cd "$(dirname "$0")/.."
T=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="paper_2302_04852_b200/build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/${T}_ab.log
  for t in 16384 2048; do
    SPARSEPROP_LIB=$L timeout 300 python bench.py --tokens $t --no-configs --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | grep "^{" | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(json.dumps({'tokens': $t, 'ms': d['ms_per_step'], 'e2e_gflops': d['e2e']['value']}))" >> gpurun_out/${T}_ab.log
  done
  SPARSEPROP_LIB=$L timeout 600 python tools/cfg_time.py cfg2a cfg2b cfg4:uniform:0.95 cfg4:uniform:0.99 cfg3 >> gpurun_out/${T}_ab.log 2>&1
done

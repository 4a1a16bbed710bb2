#!/bin/bash
# Round measurement on one B200 (run under gpurun): bench line, ncu launch list of a
# short bench run, ncu --set full of the top kernels.  Outputs land in gpurun_out/$TAG*.
cd "$(dirname "$0")/.."
TAG=${1:-m}
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 > gpurun_out/${TAG}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 > gpurun_out/${TAG}_ncu_launches.log 2>&1 &&
python tools/prof_layer.py --iters 1 > gpurun_out/${TAG}_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"bwd_fused|spmm_tiled|spmm_hyb" -c 6 \
    -o gpurun_out/${TAG}_full python tools/prof_layer.py --iters 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "measure rc=$?" >> gpurun_out/${TAG}_bench.log

#!/bin/bash
# Round-2 measurement on one B200 (under gpurun): the bench line, the ncu launch
# list of a short bench run, --set full captures of the cfg5 kernels (dominant:
# the fused backward), of the single-layer configs (cfg2a, cfg4 95% uniform /
# Zipf, cfg4 99%) and of cfg3.  Outputs: gpurun_out/${TAG}_*.
cd "$(dirname "$0")/.."
TAG=${1:-m2}
# reports are summarised on the box (raw metric page + per-kernel summary +
# source-page hot spots); only the cfg5 report itself is kept (gpurun copies
# back at most 64 MiB)
summ() {
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  python tools/ncu_full_summary.py gpurun_out/$1.ncu-rep > gpurun_out/$1_summary.txt 2>&1
  python tools/ncu_traffic.py gpurun_out/$1.ncu-rep gpurun_out/$1_traffic.json "$1" > /dev/null 2>&1
  [ "$2" = keep ] || rm -f gpurun_out/$1.ncu-rep
}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
python bench.py > gpurun_out/${TAG}_bench.log 2>&1 || exit 1
# launch list (same command twice: plain first, then under ncu; eager steps: ncu cannot
# follow the whole-step graph capture -- the capture launch fails under it)
python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --graph 0 > gpurun_out/${TAG}_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --graph 0 > gpurun_out/${TAG}_ncu_launches.log 2>&1
# cfg5 layer kernels: fwd (split-source SpMM), fused backward
python tools/prof_layer.py --iters 1 > gpurun_out/${TAG}_plain2.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:spmm_hyb|bwd_fused' -c 4 \
    -o gpurun_out/${TAG}_full_cfg5 python tools/prof_layer.py --iters 1 > gpurun_out/${TAG}_ncu_cfg5.log 2>&1
summ ${TAG}_full_cfg5 keep
# single-layer configs: fwd SpMM, dX SpMM, dW alone, fused backward
for a in "0.95 uniform" "0.95 zipf" "0.99 uniform"; do
  set -- $a
  python tools/prof_cfg4.py --sparsity $1 --kind $2 --iters 1 > gpurun_out/${TAG}_plain_$2$1.log 2>&1 &&
  timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:spmm|bwd_fused|gather' -c 4 \
      -o gpurun_out/${TAG}_full_cfg4_$2$1 python tools/prof_cfg4.py --sparsity $1 --kind $2 --iters 1 \
      > gpurun_out/${TAG}_ncu_cfg4_$2$1.log 2>&1
  summ ${TAG}_full_cfg4_$2$1
done
python tools/prof_layer.py --B 512 --iters 1 > gpurun_out/${TAG}_plain3.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:spmm|bwd_fused' -c 4 \
    -o gpurun_out/${TAG}_full_cfg2a python tools/prof_layer.py --B 512 --iters 1 > gpurun_out/${TAG}_ncu_cfg2a.log 2>&1
summ ${TAG}_full_cfg2a
python tools/prof_conv.py --iters 1 > gpurun_out/${TAG}_plain4.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:spmm|bwd_fused|sddmm' -c 4 \
    -o gpurun_out/${TAG}_full_cfg3 python tools/prof_conv.py --iters 1 > gpurun_out/${TAG}_ncu_cfg3.log 2>&1
summ ${TAG}_full_cfg3
echo "measure done" >> gpurun_out/${TAG}_bench.log

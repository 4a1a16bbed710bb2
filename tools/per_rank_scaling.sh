#!/bin/bash
# One B200 running one rank's token share of a 1/2/4/8-GPU strong-scaling run
# (bench.py --tokens T: graph-replayed step, no all_reduce) -> gpurun_out/${TAG}_per_rank.jsonl
cd "$(dirname "$0")/.."
TAG=${1:-pr}
OUT=gpurun_out/${TAG}_per_rank.jsonl
: > $OUT
for t in 16384 8192 4096 2048; do
  timeout 600 python bench.py --tokens $t --no-configs --no-cpu-baseline --steps 20 --warmup 5 2>/dev/null | grep "^{" |
  python -c "
import sys, json
d = json.loads(sys.stdin.readline())
print(json.dumps({'tokens': $t, 'ms_per_step': d['ms_per_step'], 'gflops': d['value'], 'e2e_gflops': d['e2e']['value'],
                  'launches_per_step': d['gpu_launches'] / d['steps'], 'clocks': d['clocks'], 'ranks': 16384 // $t}))" >> $OUT
done
python - $OUT <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1])]
t1 = rows[0]['ms_per_step']
with open(sys.argv[1], 'w') as f:
    for r in rows:
        r['per_rank_efficiency_before_allreduce'] = round(t1 / (r['ranks'] * r['ms_per_step']), 4)
        r['note'] = "one B200 running one rank's token share of a strong-scaling run (bench.py --tokens T, graph-replayed step, no all_reduce)"
        f.write(json.dumps(r) + "\n")
PY

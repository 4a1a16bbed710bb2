#!/bin/bash
# per-tile row balancing (refine_rows) A/B: cfg5 layer kernels and handle-creation time
cd "$(dirname "$0")/.."
for m in "SP_ROW_REFINE=0" ""; do
  echo "== $m" >> gpurun_out/ab_refine.log
  (env $m timeout 120 python tools/prof_layer.py; env $m timeout 120 python tools/prof_layer.py --R 768 --C 3072; env $m timeout 120 python tools/prof_layer.py --B 2048) 2>&1 | grep -E "fwd|fused" | tr '\n' ' ' >> gpurun_out/ab_refine.log
  echo >> gpurun_out/ab_refine.log
  env $m timeout 120 python - >> gpurun_out/ab_refine.log 2>&1 <<'PY'
import time, torch, synth
from paper_2302_04852_b200 import sparseprop as sp
c = synth.linear_case(3072, 768, 8, 0.05, 1.0 / 768, 5)
W, M = torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda()
sp.sp_weight_create(W, M); torch.cuda.synchronize()
t = time.time(); [sp.sp_weight_create(W, M) for _ in range(5)]; torch.cuda.synchronize()
print(f"sp_weight_create 3072x768 d=0.05: {(time.time() - t) / 5 * 1e3:.1f} ms")
PY
done
timeout 300 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/refine_tests.log 2>&1; echo rc=$? >> gpurun_out/refine_tests.log

#!/bin/bash
# per-kernel layer timings for several env settings: tools/ab_env.sh "SP_X=1" "SP_Y=2 SP_Z=0" ...
cd "$(dirname "$0")/.."
for args in "" "--R 768 --C 3072" "--B 2048" "--R 4096 --C 4096 --B 256 --density 0.1"; do
  echo "== $args"
  python tools/prof_layer.py $args | grep -E "bwd_fused|dw" | sed "s/^/base  /"
  for e in "$@"; do env $e python tools/prof_layer.py $args | grep -E "bwd_fused|dw" | sed "s/^/$e  /"; done
done

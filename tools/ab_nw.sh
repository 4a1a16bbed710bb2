cd /root/repo
for args in "" "--R 768 --C 3072" "--B 2048" "--R 4096 --C 4096 --B 256 --density 0.1"; do
  echo "== $args"
  for nw in 32 28 24 16; do SP_FUSED_NW=$nw python tools/prof_layer.py $args | grep bwd_fused | sed "s/^/NW$nw /"; done
done

"""Time the conv hot path (cfg3 shapes by default) per product, CUDA events, one call each."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
c = synth.conv_case(**synth.CFG["cfg3"])
W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
g = sp.conv_geom(W, c["B"], c["H"], c["Wd"], c["pad"])
X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
Y = torch.empty(c["OC"], c["OH"], c["OW"], c["B"], device="cuda")
dX = torch.empty_like(X)
dW = torch.empty(W.nnz, device="cuda")
res = {}
for it in range(args.iters):
    for name, f in (("fwd", lambda: sp.sp_conv2d_fwd(W, g, X, Y)), ("dx", lambda: sp.sp_conv2d_bwd_input(W, g, dY, dX)),
                    ("dw", lambda: sp.sp_conv2d_bwd_weight(W, g, X, dY, dW)),
                    ("bwd_fused", lambda: sp.sp_conv2d_bwd(W, g, X, dY, dX, dW))):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        res.setdefault(name, []).append(s.elapsed_time(e))
for k, v in res.items():
    print(f"conv {k}: {min(v)*1e3:.1f} us")

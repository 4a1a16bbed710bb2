"""Time the cfg4 products (fwd, dX, dW, fused backward) for one sparsity and
mask kind with CUDA events (no L2 flush; quick A/B of kernel choices through
the SP_* environment switches).  Also prints the mask's row-length profile."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sparsity", type=float, default=0.99)
ap.add_argument("--kind", default="zipf")
ap.add_argument("--iters", type=int, default=5)
args = ap.parse_args()
cf = synth.cfg4(args.sparsity, args.kind)
c = synth.linear_case(cf["R"], cf["C"], cf["B"], cf["density"], cf["wvar"], cf["seed"], cf["kind"])
rl = np.sort(c["mask"].sum(1))[::-1]
print(f"cfg4 {args.kind} {args.sparsity}: nnz {int(rl.sum())}, longest rows {rl[:6].tolist()}, median {int(np.median(rl))}")
W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
X = torch.from_numpy(c["X"]).cuda()
dY = torch.from_numpy(c["dY"]).cuda()
Y = torch.empty(cf["R"], cf["B"], device="cuda")
dX = torch.empty(cf["C"], cf["B"], device="cuda")
dW = torch.empty(W.nnz, device="cuda")
res = {}
for it in range(args.iters):
    for name, f in (("fwd", lambda: sp.sp_linear_fwd(W, X, Y)), ("dx", lambda: sp.sp_linear_bwd_input(W, dY, dX)),
                    ("dw", lambda: sp.sp_linear_bwd_weight(W, X, dY, dW)),
                    ("bwd_fused", lambda: sp.sp_linear_bwd(W, X, dY, dX, dW))):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        res.setdefault(name, []).append(s.elapsed_time(e))
print("  ".join(f"{k} {1e3 * min(v):.1f} us" for k, v in res.items()))

"""Run each linear hot-path kernel once per iteration on cfg5-shaped layers
(for ncu captures and quick per-kernel CUDA-event timings)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=16384)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--R", type=int, default=3072)
ap.add_argument("--C", type=int, default=768)
ap.add_argument("--density", type=float, default=0.05)
args = ap.parse_args()

c = synth.linear_case(args.R, args.C, args.B, args.density, 1.0 / args.C, 5)
W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
X = torch.from_numpy(c["X"]).cuda()
dY = torch.from_numpy(c["dY"]).cuda()
Y = torch.empty(args.R, args.B, device="cuda")
dX = torch.empty(args.C, args.B, device="cuda")
dW = torch.empty(W.nnz, device="cuda")
fl = 2 * W.nnz * args.B
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
for k, v in res.items():
    t = min(v)
    f = fl * (2 if k == "bwd_fused" else 1)
    print(f"{k}: {t*1e3:.1f} us  {f / (t*1e-3) / 1e12:.2f} TFLOP/s  ({f/(t*1e-3)/1e12/74.45*100:.1f}% of FP32 peak)")

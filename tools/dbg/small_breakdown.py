"""Measurement only: the kernels of one fwd + fused bwd call of a small-batch
layer (default cfg2a), for an ncu launch list (python tools/dbg/small_breakdown.py
under ncu --metrics gpu__time_duration.sum) and CUDA-event times of each call."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2a")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
if a.cfg.startswith("cfg4:"):  # cfg4:sparsity:kind
    _, s_, kind = a.cfg.split(":")
    c4 = synth.cfg4(float(s_), kind)
    cf = dict(R=c4["R"], C=c4["C"], B=c4["B"], density=c4["density"], wvar=c4["wvar"], seed=c4["seed"], kind=kind)
else:
    cf = synth.CFG[a.cfg]
if a.cfg == "cfg3":
    c = synth.conv_case(**cf)
    W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
    g = sp.conv_geom(W, c["B"], c["H"], c["Wd"], c["pad"])
    Y = torch.empty(c["OC"], c["OH"], c["OW"], c["B"], device="cuda")
else:
    c = synth.linear_case(**cf)
    R, C, B = cf["R"], cf["C"], cf["B"]
    W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
    Y = torch.empty(R, B, device="cuda")
sp.sp_weight_set_managed(W, True)
X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
dX = torch.empty_like(X)
dW = torch.empty(W.nnz, device="cuda")
flush = torch.empty(64 << 20, device="cuda")
if a.cfg == "cfg3":
    calls = (("fwd", lambda: sp.sp_conv2d_fwd(W, g, X, Y)), ("bwd", lambda: sp.sp_conv2d_bwd(W, g, X, dY, dX, dW)))
else:
    calls = (("fwd", lambda: sp.sp_linear_fwd(W, X, Y)), ("bwd", lambda: sp.sp_linear_bwd(W, X, dY, dX, dW)))
for it in range(a.iters):
    for name, f in calls:
        flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        print(it, name, f"{s.elapsed_time(e) * 1e3:.1f} us", sp.last_path())

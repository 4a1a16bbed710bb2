"""Measurement only: forward time of the cfg5 layer shapes vs batch (wave
quantisation of the per-item grid: 768-row layer = 6 row blocks x B/128 slices)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402

for R, C in ((768, 3072), (3072, 768)):
    c = synth.linear_case(R, C, 128, 0.05, 1.0 / C, 5)
    W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
    sp.sp_weight_set_managed(W, True)
    for B in (14208, 15744, 15872, 16000, 16384):
        X = torch.randn(C, B, device="cuda")
        Y = torch.empty(R, B, device="cuda")
        for _ in range(3):
            sp.sp_linear_fwd(W, X, Y)
        ts = []
        for _ in range(7):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            sp.sp_linear_fwd(W, X, Y)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        items = ((R + 127) // 128) * (B // 128)
        print(f"{R}x{C} B={B} items={items} waves={items / 148:.2f} fwd {ts[3]:.1f} us  per-slice {ts[3] / (B // 128):.3f} us  {sp.last_path()}")

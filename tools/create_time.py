"""sp_weight_create wall time (host, synchronised) for the BASELINE layer shapes:
median of 5 creations after one warm-up (allocator / module load excluded)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402


def t_create(W, M, n=5):
    sp.sp_weight_create(W, M)
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        h = sp.sp_weight_create(W, M)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del h
    ts.sort()
    return ts[len(ts) // 2] * 1e3


recs = []
for name, (R, C, d) in {"cfg5_W1 3072x768": (3072, 768, 0.05), "cfg5_W2 768x3072": (768, 3072, 0.05),
                        "cfg4 4096^2 95%": (4096, 4096, 0.05), "cfg4 4096^2 80%": (4096, 4096, 0.2),
                        "cfg4 4096^2 99% (+ gather tilings)": (4096, 4096, 0.01),
                        "cfg1 256^2 90% (+ gather tilings)": (256, 256, 0.1)}.items():
    c = synth.linear_case(R, C, 4, d, 1.0 / C, 7)
    recs.append({"shape": name, "nnz": int(c["mask"].sum()),
                 "create_ms": round(t_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda()), 3)})
cc = synth.conv_case(**synth.CFG["cfg3"])
recs.append({"shape": "cfg3 conv 256x256x3x3 90%", "nnz": int(cc["mask"].sum()),
             "create_ms": round(t_create(torch.from_numpy(cc["W"]).cuda(), torch.from_numpy(cc["mask"]).cuda()), 3)})
for r in recs:
    print(json.dumps(r))

"""Per-CTA timeline of one fused-backward launch (measurement build with
SP_FUSED_TS: tools/build_variant.py fts SP_FUSED_TS; SPARSEPROP_LIB=...fts.so)."""
import ctypes as ct
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402

R, C, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
c = synth.linear_case(R, C, B, 0.05, 1.0 / C, 5)
W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
sp.sp_weight_set_managed(W, True)
X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
dX = torch.empty(C, B, device="cuda")
dW = torch.empty(W.nnz, device="cuda")
for _ in range(5):
    sp.sp_linear_bwd(W, X, dY, dX, dW)
torch.cuda.synchronize()
L = sp.lib()
f = L.sp_debug_fused_ts
f.restype, f.argtypes = ct.c_int, [ct.c_void_p, ct.c_int]
buf = np.zeros((1024, 4), dtype=np.uint64)
assert f(buf.ctypes.data, 1024) == 0
ts = buf[:148].astype(np.int64)
t0 = ts[:, 0].min()
ts = (ts - t0) / 1e3  # us
print(f"{R}x{C} B={B} path={sp.last_path()}")
for k, name in enumerate(["entry", "first tile", "loop done", "exit"]):
    col = ts[:, k]
    print(f"  {name:10s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us")
print(f"  prologue (first tile - entry) med {np.median(ts[:,1]-ts[:,0]):.2f} max {(ts[:,1]-ts[:,0]).max():.2f}")
print(f"  loop (loop done - first tile) min {(ts[:,2]-ts[:,1]).min():.2f} med {np.median(ts[:,2]-ts[:,1]):.2f} max {(ts[:,2]-ts[:,1]).max():.2f}")
print(f"  epilogue (exit - loop done) med {np.median(ts[:,3]-ts[:,2]):.2f} max {(ts[:,3]-ts[:,2]).max():.2f}")

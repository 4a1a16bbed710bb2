import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth
from paper_2302_04852_b200 import sparseprop as sp
R, C, B, d = [float(x) if '.' in x else int(x) for x in sys.argv[1:5]]
op = sys.argv[5]
c = synth.linear_case(R, C, B, d, 1.0 / C, 1)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
W = sp.sp_weight_create(dev(c["W"]), dev(c["mask"]))
X, dY = dev(c["X"]), dev(c["dY"])
if op == "dw": o = sp.sp_linear_bwd_weight(W, X, dY)
elif op == "bwd": o = sp.sp_linear_bwd(W, X, dY)[1]
else: o = sp.sp_linear_fwd(W, X)
print(sp.last_path(), flush=True)
torch.cuda.synchronize()
print("ok", float(o.abs().sum()))

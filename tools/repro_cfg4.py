import sys, os, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2302_04852_b200 import sparseprop as sp
cf = synth.cfg4(float(sys.argv[1]), sys.argv[2])
c = synth.linear_case(cf["R"], cf["C"], cf["B"], cf["density"], cf["wvar"], cf["seed"], sys.argv[2])
W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
for name, f in (("fwd", lambda: sp.sp_linear_fwd(W, X)), ("dx", lambda: sp.sp_linear_bwd_input(W, dY)),
                ("dw", lambda: sp.sp_linear_bwd_weight(W, X, dY)), ("fused", lambda: sp.sp_linear_bwd(W, X, dY))):
    f(); torch.cuda.synchronize(); print(name, "ok", flush=True)

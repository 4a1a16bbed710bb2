import sys, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2302_04852_b200 import sparseprop as sp
def dev(a): return torch.from_numpy(a).cuda()
for (R, C, B, d) in [(3072, 768, 512, 0.05), (500, 300, 200, 0.1), (1024, 512, 256, 0.2)]:
    c = synth.linear_case(R, C, B, d, 1.0 / C, 3)
    W = sp.sp_weight_create(dev(c["W"]), dev(c["mask"]))
    X, dY = dev(c["X"]), dev(c["dY"])
    sp.sp_linear_fwd(W, X); sp.sp_linear_bwd(W, X, dY); sp.sp_linear_bwd_weight(W, X, dY); sp.sp_linear_bwd_input(W, dY)
    torch.cuda.synchronize(); print("linear", R, C, B, d, "ok", flush=True)
cc = synth.conv_case(OC=64, IC=32, H=8, W=8, KH=3, KW=3, pad=1, B=16, density=0.2, wvar=1.0 / 288, seed=5)
Wc = sp.sp_weight_create(dev(cc["W"]), dev(cc["mask"]))
g = sp.conv_geom(Wc, 16, 8, 8, 1)
Xc, dYc = dev(cc["X"]), dev(cc["dY"])
sp.sp_conv2d_fwd(Wc, g, Xc); sp.sp_conv2d_bwd(Wc, g, Xc, dYc); torch.cuda.synchronize(); print("conv ok", flush=True)

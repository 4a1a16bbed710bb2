"""GPU parity of every A/B kernel switch (README "A/B switches") against the
fp64 oracle: the split-source and TMEM-gather SpMMs, the stream-K / per-item
SpMM choice, the 16-warp SpMM, and the fused-backward and conv variants.  The
switches are read once per process, so every setting runs in its own
interpreter on the same seeded cases: fwd (+ ReLU), dX, the fused backward
(dX and dW) and a conv forward / fused backward."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch, oracle, synth
from conftest import tol_ok
from paper_2302_04852_b200 import sparseprop as sp

def ok(name, got, ref):
    good, err, bound = tol_ok(got, ref)
    assert good, (name, err, bound)

cases = [synth.linear_case(**synth.CFG["cfg2a"]), synth.linear_case(**synth.CFG["cfg2b"]),
         synth.linear_case(601, 397, 516, 0.1, 1.0 / 397, 77),   # ragged rows / columns / batch tail
         synth.linear_case(512, 640, 256, 0.05, 1.0 / 640, 78, "zipf"),
         synth.linear_case(3072, 768, 2048, 0.05, 1.0 / 768, 79)]
for c in cases:
    W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
    X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
    Y = sp.sp_linear_fwd(W, X).cpu().numpy()
    Yr = sp.sp_linear_fwd(W, X, relu=True).cpu().numpy()
    dX = sp.sp_linear_bwd_input(W, dY).cpu().numpy()
    fdX, fdW = (t.cpu().numpy() for t in sp.sp_linear_bwd(W, X, dY))
    S = oracle.csr_from_mask(c["W"], c["mask"])
    ref = oracle.linear_fwd(S, c["X"], 8)
    refx = oracle.linear_bwd_input(S, c["dY"], 8)
    ok("Y", Y, ref)
    ok("relu(Y)", Yr, np.maximum(ref, 0.0))
    ok("dX", dX, refx)
    ok("fused dX", fdX, refx)
    ok("fused dW", fdW, oracle.linear_bwd_weight(S, c["X"], c["dY"], 8))
cc = synth.conv_case(**synth.CFG["cfg3"])
Wc = sp.sp_weight_create(torch.from_numpy(cc["W"]).cuda(), torch.from_numpy(cc["mask"]).cuda())
g = sp.conv_geom(Wc, cc["B"], cc["H"], cc["Wd"], cc["pad"])
Xc, dYc = torch.from_numpy(cc["X"]).cuda(), torch.from_numpy(cc["dY"]).cuda()
Yc = sp.sp_conv2d_fwd(Wc, g, Xc).cpu().numpy()
dXc, dWc = (t.cpu().numpy() for t in sp.sp_conv2d_bwd(Wc, g, Xc, dYc))
F = oracle.conv_format(cc["W"], cc["mask"])
Xn, dOn = oracle.chwn_to_nchw(cc["X"]), oracle.chwn_to_nchw(cc["dY"])
ok("conv Y", Yc, oracle.nchw_to_chwn(oracle.conv2d_fwd(F, Xn, cc["pad"], 8)))
rdX, rdW = oracle.conv2d_bwd(F, Xn, dOn, cc["pad"])
ok("conv dX", dXc, oracle.nchw_to_chwn(rdX))
ok("conv dW", dWc, rdW)
print("ok")
"""

SWITCHES = {
    "default": {},
    "spmm_sk0": dict(SP_SPMM_SK="0"),
    "spmm_sk1": dict(SP_SPMM_SK="1"),
    "spmm_nw16": dict(SP_SPMM_NW32="0"),
    "spmm_rb256": dict(SP_SPMM_RB256="1"),
    "hyb": dict(SP_SPMM_HYB="1"),
    "hyb_off": dict(SP_SPMM_HYB="0"),
    "tm0": dict(SP_SPMM_TM="1", SP_SPMM_TM_VAR="0"),
    "tm1": dict(SP_SPMM_TM="1", SP_SPMM_TM_VAR="1"),
    "tm2": dict(SP_SPMM_TM="1", SP_SPMM_TM_VAR="2"),
    "tm3": dict(SP_SPMM_TM="1", SP_SPMM_TM_VAR="3"),
    "fused_whole_warp": dict(SP_FUSED_HALF="0"),
    "fused_nw16": dict(SP_FUSED_NW="16"),
    "fused_nw24": dict(SP_FUSED_NW="24"),
    "fused_nw28": dict(SP_FUSED_NW="28"),
    "fused_no_sk": dict(SP_FUSED_SK="0"),
    "fused_kc128": dict(SP_FUSED_KC128="1"),
    "fused_no_tmem": dict(SP_FUSED_TMEM="0"),
    "conv_no_sk": dict(SP_CONV_SK="0"),
    "gather_on": dict(SP_GATHER="1"),
    "gather_off": dict(SP_GATHER="0"),
}


@pytest.mark.parametrize("name", list(SWITCHES))
def test_switch_matches_oracle(name):
    env = dict(os.environ, **SWITCHES[name])
    env["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), env.get("PYTHONPATH", "")])
    p = subprocess.run([sys.executable, "-c", SCRIPT], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert "ok" in p.stdout

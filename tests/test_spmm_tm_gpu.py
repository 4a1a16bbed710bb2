"""GPU parity of the SpMM kernels that gather from tensor memory against the
fp64 oracle: the split-source SpMM (spmm_hyb.cu, SP_SPMM_HYB=1) and each CTA
layout of the opt-in TMEM-gather SpMM (spmm_tm.cu, SP_SPMM_TM=1,
SP_SPMM_TM_VAR).  The switches are read once per process, so every setting
runs in its own interpreter."""
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
cases = [synth.linear_case(**synth.CFG["cfg2a"]), synth.linear_case(**synth.CFG["cfg2b"]),
         synth.linear_case(601, 397, 516, 0.1, 1.0 / 397, 77),   # ragged rows / columns / batch tail
         synth.linear_case(512, 640, 256, 0.05, 1.0 / 640, 78, "zipf")]
for c in cases:
    W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
    X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
    Y = sp.sp_linear_fwd(W, X).cpu().numpy()
    Yr = sp.sp_linear_fwd(W, X, relu=True).cpu().numpy()
    dX = sp.sp_linear_bwd_input(W, dY).cpu().numpy()
    S = oracle.csr_from_mask(c["W"], c["mask"])
    ref = oracle.linear_fwd(S, c["X"], 8)
    for name, got, r in (("Y", Y, ref), ("relu(Y)", Yr, np.maximum(ref, 0.0)),
                         ("dX", dX, oracle.linear_bwd_input(S, c["dY"], 8))):
        ok, err, bound = tol_ok(got, r)
        assert ok, (c["W"].shape, name, err, bound)
print("ok", sp.launch_count() if hasattr(sp, "launch_count") else "")
"""


@pytest.mark.parametrize("switch", [dict(SP_SPMM_HYB="1")] +
                         [dict(SP_SPMM_TM="1", SP_SPMM_TM_VAR=str(v)) for v in range(4)],
                         ids=["hyb", "tm0", "tm1", "tm2", "tm3"])
def test_tmem_spmm_matches_oracle(switch):
    env = dict(os.environ, **switch)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), env.get("PYTHONPATH", "")])
    p = subprocess.run([sys.executable, "-c", SCRIPT], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert "ok" in p.stdout

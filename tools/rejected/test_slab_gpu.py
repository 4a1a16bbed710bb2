"""The batch-slab kernels (csrc/slab.cu): the very sparse regime's products
from a shared-memory slab of the whole inner dimension of a narrow batch slice
-- forward, dX, dW alone and the fused backward (plain and ReLU'-gated), every
slab width (8 / 16 / 32 / 64 columns, chosen by the inner dimension), ragged
last slices, Zipf part rows -- against the fp64 oracle at the north-star
tolerance (PAPER.md P153-P154 CSR products, P173/P183 the single-pass
backward).  sp_last_path must name the slab kernel for each product."""
import numpy as np
import pytest

import oracle
import synth
from conftest import tol_ok

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NT = min(8, oracle.threads_available())


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2302_04852_b200 import _build, sparseprop
    _build.build()
    return sparseprop


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _ok(name, got, ref):
    ok, err, bound = tol_ok(got.detach().cpu().numpy(), ref)
    assert ok, f"{name}: max|err| {err:.3e} > {bound:.3e}"


# (R, C, B, density, kind): slab widths by inner dimension (fwd inner = C, dX inner = R)
CASES = [
    (4096, 4096, 256, 0.01, "uniform"),   # cfg4 99 % shape: 8-column slabs both ways
    (4096, 4096, 256, 0.02, "zipf"),      # cfg4 98 % Zipf: forward part rows
    (3000, 1500, 100, 0.02, "uniform"),   # fwd 32-column slabs, ragged last slice (4 of 32 columns)
    (700, 2900, 36, 0.02, "uniform"),     # fwd 16 columns, dX 32 columns (B < 64), ragged
    (640, 600, 520, 0.03, "uniform"),     # 64-column slabs, 9 slices (last 8 columns)
    (1000, 3000, 8, 0.02, "zipf"),        # B = 8: one 8-column slice
]


@pytest.mark.parametrize("R,C,B,d,kind", CASES)
def test_slab_products(sp, R, C, B, d, kind):
    c = synth.linear_case(R, C, B, d, 1.0 / C, 31 * R + C + B, kind=kind)
    S = oracle.csr_from_mask(c["W"], c["mask"])
    W = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    X, dY = _dev(c["X"]), _dev(c["dY"])
    g = synth.rng(R + B)
    gate = synth.normal(g, (C, B), 1.0)
    gate[g.random((C, B)) < 0.3] = 0.0
    tag = f"{R}x{C} B={B} d={d} {kind}"
    rdX = oracle.linear_bwd_input(S, c["dY"], NT)
    rdW = oracle.linear_bwd_weight(S, c["X"], c["dY"], NT)
    rY = oracle.linear_fwd(S, c["X"], NT)
    runs = [
        ("fwd", lambda: [sp.sp_linear_fwd(W, X)], [rY], "spmm_slab"),
        ("fwd relu", lambda: [sp.sp_linear_fwd_relu(W, X)], [np.maximum(rY, 0.0)], "spmm_slab"),
        ("dx", lambda: [sp.sp_linear_bwd_input(W, dY)], [rdX], "spmm_slab"),
        ("dx relu'", lambda: [sp.sp_linear_bwd_input_relu(W, dY, _dev(gate))], [rdX * (gate > 0)], "spmm_slab"),
        ("dw", lambda: [sp.sp_linear_bwd_weight(W, X, dY)], [rdW], "sddmm_slab"),
        ("bwd", lambda: list(sp.sp_linear_bwd(W, X, dY)), [rdX, rdW], "bwd_slab"),
        ("bwd relu'", lambda: list(sp.sp_linear_bwd_relu(W, X, dY, _dev(gate))), [rdX * (gate > 0), rdW], "bwd_slab"),
    ]
    for name, f, refs, fam in runs:
        out = f()
        path = sp.last_path()
        torch.cuda.synchronize()
        assert fam in path.split("+"), f"{tag} {name}: expected {fam}, ran {path}"
        for o, r in zip(out, refs):
            _ok(f"{tag} {name} [{path}]", o, r)
        again = f()
        torch.cuda.synchronize()
        for o, o2 in zip(out, again):  # fixed-order sums: bitwise reproducible
            assert torch.equal(o, o2), f"{tag} {name}: not bitwise reproducible"


def test_slab_dw_exactly_zero_off_mask(sp):
    """dW from the slab's per-slice shares, densified: +0.0 off the mask."""
    c = synth.linear_case(2048, 2048, 256, 0.01, 1.0 / 2048, 77)
    W = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    dX, dW = sp.sp_linear_bwd(W, _dev(c["X"]), _dev(c["dY"]))
    assert "bwd_slab" in sp.last_path().split("+")
    D = sp.sp_weight_to_dense(W, dW, torch.empty(2048, 2048, device="cuda")).cpu().numpy()
    off = ~c["mask"].astype(bool)
    assert np.all(D[off] == 0.0) and not np.any(np.signbit(D[off]))

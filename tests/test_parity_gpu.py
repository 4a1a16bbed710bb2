"""GPU parity: libsparseprop (through its C ABI) vs the fp64 oracle on the same
seeded inputs.  Index structure bit-exact; fp32 values within the north-star
bar max|err| <= 1e-4 * max|ref| + 1e-6 per output tensor."""
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


def _np(t):
    return t.detach().cpu().numpy()


def _assert_tol(name, got, ref):
    ok, err, bound = tol_ok(got, ref)
    assert ok, f"{name}: max|err| {err:.3e} > bound {bound:.3e}"


def check_linear(sp, W, mask, X, dY, tag=""):
    """Run fwd / dX / dW on the GPU and compare everything with the oracle."""
    Wg = sp.sp_weight_create(_dev(W), _dev(mask))
    Xg, dYg = _dev(X), _dev(dY)
    Y = sp.sp_linear_fwd(Wg, Xg)
    dX = sp.sp_linear_bwd_input(Wg, dYg)
    dW = sp.sp_linear_bwd_weight(Wg, Xg, dYg)
    torch.cuda.synchronize()
    S = oracle.csr_from_mask(W, mask)
    idx = {k: _np(v) for k, v in Wg.indices().items()}
    # structure: bit-exact
    assert Wg.nnz == S.nnz, tag
    for k, ref in (("row_ptr", S.row_ptr), ("col_idx", S.col_idx), ("col_ptr", S.col_ptr),
                   ("row_idx", S.row_idx), ("perm", S.perm)):
        assert np.array_equal(idx[k], ref), f"{tag} {k}"
    assert np.array_equal(_np(Wg.vals), S.vals.astype(np.float32)), tag
    if S.nnz:
        ones = sp.sp_weight_to_dense(Wg, torch.ones(S.nnz, device="cuda"),
                                     torch.empty(W.shape, device="cuda"))
        assert np.array_equal(_np(ones) != 0, mask != 0), tag
    # values
    _assert_tol(f"{tag} Y", _np(Y), oracle.linear_fwd(S, X, NT))
    _assert_tol(f"{tag} dX", _np(dX), oracle.linear_bwd_input(S, dY, NT))
    refW = oracle.linear_bwd_weight(S, X, dY, NT)
    _assert_tol(f"{tag} dW", _np(dW), refW)
    # densified dW: exactly +0.0 off the mask
    if S.nnz:
        D = _np(Wg.to_dense(dW))
        off = D[mask == 0]
        assert np.all(off == 0.0) and not np.any(np.signbit(off)), tag
    return Wg, Y, dX, dW


# ---------------------------------------------------------------- configs
def test_cfg1(sp):
    c = synth.linear_case(**synth.CFG["cfg1"])
    check_linear(sp, c["W"], c["mask"], c["X"], c["dY"], "cfg1")


@pytest.mark.parametrize("name", ["cfg2a", "cfg2b"])
def test_cfg2(sp, name):
    c = synth.linear_case(**synth.CFG[name])
    check_linear(sp, c["W"], c["mask"], c["X"], c["dY"], name)


@pytest.mark.parametrize("kind", ["uniform", "zipf"])
@pytest.mark.parametrize("sparsity", synth.CFG4_SPARSITIES)
def test_cfg4(sp, sparsity, kind):
    cfg = synth.cfg4(sparsity, kind)
    c = synth.linear_case(cfg["R"], cfg["C"], cfg["B"], cfg["density"], cfg["wvar"], cfg["seed"], kind)
    check_linear(sp, c["W"], c["mask"], c["X"], c["dY"], f"cfg4 {kind} {sparsity}")


def _fused_vs_oracle(sp, c, tag, gate_seed=None):
    """sp_linear_bwd[_relu] (the fused backward the DP step and modules ship)
    against the oracle; returns the kernel path it took (sp_last_path)."""
    S = oracle.csr_from_mask(c["W"], c["mask"])
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    H = None
    if gate_seed is not None:
        H = synth.normal(synth.rng(gate_seed), c["X"].shape, 1.0)
        H[H < 0] = 0.0
    dX, dW = sp.sp_linear_bwd(Wg, _dev(c["X"]), _dev(c["dY"]), H=None if H is None else _dev(H))
    path = sp.last_path()
    torch.cuda.synchronize()
    refx = oracle.linear_bwd_input(S, c["dY"], NT)
    if H is not None:
        refx = refx * (H > 0)
    _assert_tol(f"{tag} fused dX [{path}]", _np(dX), refx)
    _assert_tol(f"{tag} fused dW [{path}]", _np(dW), oracle.linear_bwd_weight(S, c["X"], c["dY"], NT))
    return path


@pytest.mark.parametrize("kind", ["uniform", "zipf"])
@pytest.mark.parametrize("sparsity", synth.CFG4_SPARSITIES)
def test_cfg4_fused_backward(sp, sparsity, kind):
    """the fused backward on every cfg4 mask (the exact
    synth.cfg4 seeds), gated and ungated, with the kernel path recorded."""
    cfg = synth.cfg4(sparsity, kind)
    c = synth.linear_case(cfg["R"], cfg["C"], cfg["B"], cfg["density"], cfg["wvar"], cfg["seed"], kind)
    p0 = _fused_vs_oracle(sp, c, f"cfg4 {kind} {sparsity}")
    p1 = _fused_vs_oracle(sp, c, f"cfg4 {kind} {sparsity} gated", gate_seed=cfg["seed"] + 1)
    assert p0 and p1, "no kernel path recorded"
    print(f"cfg4 {kind} {sparsity}: {p0} / gated {p1}")


@pytest.mark.parametrize("name", ["cfg2a", "cfg2b"])
def test_cfg2_fused_backward(sp, name):
    c = synth.linear_case(**synth.CFG[name])
    p0 = _fused_vs_oracle(sp, c, name)
    p1 = _fused_vs_oracle(sp, c, f"{name} gated", gate_seed=77)
    assert p0 and p1
    print(f"{name}: {p0} / gated {p1}")


def test_paper_shape_B902(sp):
    # P366: (M,N) = (768, 3072), (B,M) = (902, 768); B not a multiple of 4 (S75)
    c = synth.linear_case(3072, 768, 902, 0.1, 1.0 / 768, 990)
    check_linear(sp, c["W"], c["mask"], c["X"], c["dY"], "paper B=902")


@pytest.mark.parametrize("sparsity", synth.CFG4_SPARSITIES)
def test_paper_shape_sweep_B902(sp, sparsity):
    """SURVEY §8(d) context row: the paper's Fig. 3 layer (P366: (M,N) = (768,
    3072), B = 902 -- not a multiple of 4, S75) over the 80-99 % sweep, seeds
    900 + s: structure bit-exact, fwd / dX / dW and the public fused backward
    (which takes the separate kernels' tail path here) against the oracle."""
    s100 = int(round(sparsity * 100))
    c = synth.linear_case(3072, 768, 902, 1.0 - sparsity, 1.0 / 768, 900 + s100)
    check_linear(sp, c["W"], c["mask"], c["X"], c["dY"], f"paper B=902 {sparsity}")
    W = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    fdX, fdW = sp.sp_linear_bwd(W, _dev(c["X"]), _dev(c["dY"]))
    torch.cuda.synchronize()
    S = oracle.csr_from_mask(c["W"], c["mask"])
    _assert_tol(f"paper B=902 {sparsity} fused dX", _np(fdX), oracle.linear_bwd_input(S, c["dY"], NT))
    _assert_tol(f"paper B=902 {sparsity} fused dW", _np(fdW), oracle.linear_bwd_weight(S, c["X"], c["dY"], NT))


@pytest.mark.parametrize("R,C,B,d", [(3072, 768, 902, 0.05), (768, 3072, 66, 0.05), (1000, 700, 201, 0.01)])
def test_padded_backward(sp, R, C, B, d):
    """B % 4 != 0 from 64 columns on: the backward runs on zero-padded copies
    (sp_last_path names pad_b4) -- ungated, ReLU'-gated by a separate H, and
    gated by X itself (the DP step's H == X, whose padded copy is reused) --
    against the oracle; the padding's zero columns must not leak into dW."""
    c = synth.linear_case(R, C, B, d, 1.0 / C, R + C + B)
    S = oracle.csr_from_mask(c["W"], c["mask"])
    W = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    X, dY = _dev(c["X"]), _dev(c["dY"])
    g = synth.rng(B)
    gate = synth.normal(g, (C, B), 1.0)
    rdX, rdW = oracle.linear_bwd_input(S, c["dY"], NT), oracle.linear_bwd_weight(S, c["X"], c["dY"], NT)
    for name, call, rx in (("plain", lambda: sp.sp_linear_bwd(W, X, dY), rdX),
                           ("gate H", lambda: sp.sp_linear_bwd_relu(W, X, dY, _dev(gate)), rdX * (gate > 0)),
                           ("gate X", lambda: sp.sp_linear_bwd_relu(W, X, dY, X), rdX * (c["X"] > 0))):
        fdX, fdW = call()
        path = sp.last_path()
        torch.cuda.synchronize()
        assert "pad_b4" in path.split("+"), path
        _assert_tol(f"padded {name} dX [{path}]", _np(fdX), rx)
        _assert_tol(f"padded {name} dW [{path}]", _np(fdW), rdW)
    dW = sp.sp_linear_bwd_weight(W, X, dY)
    assert "pad_b4" in sp.last_path().split("+")
    _assert_tol("padded dW alone", _np(dW), rdW)


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("R,C,B,d", [
    (1, 1, 1, 1.0), (1, 7, 3, 0.5), (7, 1, 5, 0.5), (37, 53, 1, 0.2), (64, 48, 33, 0.15),
    (200, 130, 3, 0.05), (129, 257, 67, 0.3), (300, 41, 130, 0.5), (96, 1500, 9, 0.02),
    (1200, 64, 200, 0.01), (40, 40, 1024, 1.0)])
def test_ragged_shapes(sp, R, C, B, d):
    c = synth.linear_case(R, C, B, d, 1.0 / C, R * 1000 + C * 10 + B)
    check_linear(sp, c["W"], c["mask"], c["X"], c["dY"], f"{R}x{C} B={B}")


def test_empty_mask(sp):
    g = synth.rng(5)
    W = synth.normal(g, (33, 17), 1.0)
    X = synth.normal(g, (17, 40), 1.0)
    dY = synth.normal(g, (33, 40), 1.0)
    Wg = sp.sp_weight_create(_dev(W), _dev(np.zeros((33, 17), np.uint8)))
    assert Wg.nnz == 0
    Y = sp.sp_linear_fwd(Wg, _dev(X), torch.full((33, 40), 7.0, device="cuda"))
    dX = sp.sp_linear_bwd_input(Wg, _dev(dY), torch.full((17, 40), 7.0, device="cuda"))
    dW = sp.sp_linear_bwd_weight(Wg, _dev(X), _dev(dY))
    torch.cuda.synchronize()
    assert np.all(_np(Y) == 0) and np.all(_np(dX) == 0) and dW.numel() == 0


def test_empty_rows_and_columns(sp):
    g = synth.rng(6)
    mask = synth.bernoulli_mask(g, 80, 70, 0.2)
    mask[5:20] = 0
    mask[:, 30:45] = 0
    W = synth.normal(g, (80, 70), 1.0 / 70)
    X = synth.normal(g, (70, 65), 1.0)
    dY = synth.normal(g, (80, 65), 1.0)
    _, Y, dX, _ = check_linear(sp, W, mask, X, dY, "empty rows/cols")
    assert np.all(_np(Y)[5:20] == 0) and np.all(_np(dX)[30:45] == 0)


def test_on_mask_zero_values_are_stored(sp):
    g = synth.rng(7)
    mask = synth.bernoulli_mask(g, 50, 60, 0.3)
    W = synth.normal(g, (50, 60), 0.1)
    W[mask.astype(bool) & (g.random((50, 60)) < 0.3)] = 0.0
    X = synth.normal(g, (60, 36), 1.0)
    dY = synth.normal(g, (50, 36), 1.0)
    Wg, *_ = check_linear(sp, W, mask, X, dY, "on-mask zeros")
    assert Wg.nnz == int(mask.sum())


# ---------------------------------------------------------------- properties
def test_bitwise_determinism_and_batch_invariance(sp):
    c = synth.linear_case(3072, 768, 512, 0.05, 1.0 / 768, 77)
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    X, dY = _dev(c["X"]), _dev(c["dY"])
    outs = [(sp.sp_linear_fwd(Wg, X), sp.sp_linear_bwd_input(Wg, dY), sp.sp_linear_bwd_weight(Wg, X, dY))
            for _ in range(2)]
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    # forward of a token is independent of the batch it is in (fixed per-element order)
    Y_sub = sp.sp_linear_fwd(Wg, X[:, :96].contiguous())
    Y_one = sp.sp_linear_fwd(Wg, X[:, 5:6].contiguous())
    torch.cuda.synchronize()
    assert torch.equal(Y_sub, outs[0][0][:, :96])
    assert torch.equal(Y_one[:, 0], outs[0][0][:, 5])


def test_fused_backward_bitwise_determinism(sp):
    """The stream-K fused backward (split items add two gated partials, dW
    partial rows summed in fixed order) gives bitwise identical results run to run."""
    c = synth.linear_case(3072, 768, 16384, 0.05, 1.0 / 768, 79)
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    X, dY = _dev(c["X"]), _dev(c["dY"])
    H = torch.relu(_dev(synth.normal(synth.rng(80), (768, 16384), 1.0)))
    outs = [sp.sp_linear_bwd(Wg, X, dY, H=H) for _ in range(3)]
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1])


def test_relu_epilogues(sp):
    c = synth.linear_case(300, 200, 70, 0.1, 1.0 / 200, 88)
    S = oracle.csr_from_mask(c["W"], c["mask"])
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    H = sp.sp_linear_fwd_relu(Wg, _dev(c["X"]))
    torch.cuda.synchronize()
    ref = np.maximum(oracle.linear_fwd(S, c["X"]), 0.0)
    _assert_tol("relu fwd", _np(H), ref)
    # gate: dX = (W^T dY) * [Hg > 0] with an arbitrary gate tensor with exact zeros
    g = synth.rng(89)
    gate = synth.normal(g, (200, 70), 1.0)
    gate[g.random((200, 70)) < 0.3] = 0.0
    dX = sp.sp_linear_bwd_input_relu(Wg, _dev(c["dY"]), _dev(gate))
    torch.cuda.synchronize()
    refx = oracle.linear_bwd_input(S, c["dY"]) * (gate > 0)
    _assert_tol("relu' dX", _np(dX), refx)
    assert np.all(_np(dX)[gate <= 0] == 0)


def test_mse_and_sgd(sp):
    g = synth.rng(90)
    Y = synth.normal(g, (768, 1000), 1.0)
    T = synth.normal(g, (768, 1000), 1.0)
    dY = torch.empty(768, 1000, device="cuda")
    loss = torch.zeros(1, device="cuda")
    scratch = torch.empty(sp.sp_mse_scratch_floats(Y.size), device="cuda")
    sp.sp_mse_grad(_dev(Y), _dev(T), dY, loss, scratch)
    torch.cuda.synchronize()
    d = Y.astype(np.float64) - T
    assert np.array_equal(_np(dY), (Y - T).astype(np.float32))
    assert float(loss) == pytest.approx(0.5 * float(np.sum(d * d)), rel=1e-6)
    v = synth.normal(g, 1000, 1.0)
    w = synth.normal(g, 1000, 1.0)
    vt = _dev(v)
    sp.sp_sgd(vt, _dev(w), 0.01)
    torch.cuda.synchronize()
    np.testing.assert_allclose(_np(vt), v.astype(np.float64) - 0.01 * w, rtol=1e-6, atol=1e-7)


# ---------------------------------------------------------------- conv
def check_conv(sp, c, tag):
    OC, IC, KH, KW, pad = c["OC"], c["IC"], c["KH"], c["KW"], c["pad"]
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    g = sp.conv_geom(Wg, c["B"], c["H"], c["Wd"], pad)
    X, dYg = _dev(c["X"]), _dev(c["dY"])
    Y = sp.sp_conv2d_fwd(Wg, g, X)
    dX = sp.sp_conv2d_bwd_input(Wg, g, dYg)
    dW = sp.sp_conv2d_bwd_weight(Wg, g, X, dYg)
    torch.cuda.synchronize()
    F = oracle.conv_format(c["W"], c["mask"])
    Xn, dOn = oracle.chwn_to_nchw(c["X"]), oracle.chwn_to_nchw(c["dY"])
    _assert_tol(f"{tag} Y", _np(Y), oracle.nchw_to_chwn(oracle.conv2d_fwd(F, Xn, pad, NT)))
    rdX, rdW = oracle.conv2d_bwd(F, Xn, dOn, pad)
    _assert_tol(f"{tag} dX", _np(dX), oracle.nchw_to_chwn(rdX))
    _assert_tol(f"{tag} dW", _np(dW), rdW)
    # both backward products in one pass (Alg. 2 single pass by taps), run twice: bitwise stable
    fused = [sp.sp_conv2d_bwd(Wg, g, X, dYg) for _ in range(2)]
    torch.cuda.synchronize()
    _assert_tol(f"{tag} fused dX", _np(fused[0][0]), oracle.nchw_to_chwn(rdX))
    _assert_tol(f"{tag} fused dW", _np(fused[0][1]), rdW)
    assert torch.equal(fused[0][0], fused[1][0]) and torch.equal(fused[0][1], fused[1][1])
    # the handle's CSR over the flattened filter is the paper's (oc, ic, x, y) order
    S = oracle.csr_from_mask(c["W"].reshape(OC, -1), c["mask"].reshape(OC, -1))
    assert np.array_equal(_np(Wg.indices()["col_idx"]), S.col_idx)
    assert Wg.nnz == F.nnz


def test_cfg3_conv(sp):
    check_conv(sp, synth.conv_case(**synth.CFG["cfg3"]), "cfg3")


def test_conv_handle_matches_linear_handle_and_is_deterministic(sp):
    c = synth.conv_case(OC=32, IC=16, H=10, W=10, KH=3, KW=3, pad=1, B=16, density=0.2, wvar=1.0 / 144, seed=77)
    Wc = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))                      # conv handle (taps)
    Wl = sp.sp_weight_create(_dev(c["W"].reshape(32, -1)), _dev(c["mask"].reshape(32, -1)))
    for k, v in Wc.indices().items():
        assert torch.equal(v, Wl.indices()[k]), k
    g = sp.conv_geom(Wc, 16, 10, 10, 1)
    X, dY = _dev(c["X"]), _dev(c["dY"])
    runs = [(sp.sp_conv2d_fwd(Wc, g, X), sp.sp_conv2d_bwd_input(Wc, g, dY), sp.sp_conv2d_bwd_weight(Wc, g, X, dY))
            for _ in range(2)]
    torch.cuda.synchronize()
    for a, b in zip(*runs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("B,IC,OC,H,W,K,pad,d", [
    (8, 4, 6, 9, 9, 7, 3, 0.3),      # 49 taps > tap-path limit -> direct kernels
    (8, 4, 6, 8, 8, 3, 3, 0.3),      # pad > K-1 -> direct kernels
    (4, 300, 140, 5, 6, 3, 1, 0.05),  # several row / column blocks on the tap path
    (3, 6, 5, 9, 9, 3, 1, 0.1), (8, 128 // 8, 256 // 8, 7, 7, 3, 1, 0.05), (2, 4, 3, 6, 5, 3, 0, 0.4),
    (1, 2, 2, 5, 5, 5, 2, 0.6), (5, 3, 2, 4, 6, 1, 0, 0.7), (33, 8, 16, 10, 10, 3, 1, 0.2),
    (64, 16, 16, 17, 19, 3, 1, 0.1), (130, 4, 4, 3, 3, 3, 1, 0.5),
    # exact-column 4-D TMA path: B > 128 (two batch slices per q), B = 128 (one q per
    # slice), partial last slices of a row (W % (128 / B) != 0), pad = K - 1, K = 5
    (256, 8, 16, 5, 6, 3, 1, 0.2), (128, 16, 8, 6, 7, 3, 2, 0.2), (32, 8, 8, 7, 7, 3, 1, 0.3),
    (16, 8, 8, 9, 7, 5, 2, 0.2), (4, 6, 6, 5, 5, 3, 0, 0.5), (64, 256, 64, 14, 14, 3, 1, 0.1),
    (12, 6, 6, 6, 6, 3, 1, 0.3),      # B does not divide 128: padded-copy fallback
])
def test_conv_shapes(sp, B, IC, OC, H, W, K, pad, d):
    c = synth.conv_case(OC=OC, IC=IC, H=H, W=W, KH=K, KW=K, pad=pad, B=B, density=d,
                        wvar=1.0 / (IC * K * K), seed=B * 7 + IC + OC + H)
    check_conv(sp, c, f"conv B={B} IC={IC} OC={OC} {H}x{W} K={K} pad={pad}")


# ---------------------------------------------------------------- fused backward (F1)
@pytest.mark.parametrize("R,C,B,d,gate", [
    (3072, 768, 2048, 0.05, False), (768, 3072, 2048, 0.05, True), (3072, 768, 16384, 0.05, True),
    (1000, 900, 384, 0.2, False),     # fused, ragged row blocks
    (300, 200, 902, 0.1, True),       # B % 4 != 0 -> separate kernels
    (200, 100, 96, 0.3, False),       # B < 128 -> separate kernels
    (64, 18944, 128, 0.05, True),     # one slice, >= 148 row blocks: dW written directly
    (2048, 256, 256, 0.5, False),     # > 4096 entries per warp: register-slot variant
    (4096, 4096, 256, 0.05, True),    # cfg4@95% shape: at the TMEM dW-column capacity of the stream-K kernel
    (3072, 768, 512, 0.05, True),     # cfg2 shape: items cut across many CTAs (last-arriver dX sums)
    (500, 300, 200, 0.1, True),       # B % 128 != 0 (a partial last slice), ragged row blocks, gated
    (4096, 1024, 256, 0.1, False),    # long CSC rows: 64-row tiling, 2 rows per warp
    (4096, 1024, 256, 0.2, True),     # longer rows: 32-row tiling, 1 row per warp
])
def test_fused_backward(sp, R, C, B, d, gate):
    c = synth.linear_case(R, C, B, d, 1.0 / C, R + C + B)
    S = oracle.csr_from_mask(c["W"], c["mask"])
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    H = None
    if gate:
        H = synth.normal(synth.rng(R + B), (C, B), 1.0)
        H[H < 0] = 0.0                      # a post-ReLU activation (exact zeros)
    dX, dW = sp.sp_linear_bwd(Wg, _dev(c["X"]), _dev(c["dY"]), H=None if H is None else _dev(H))
    torch.cuda.synchronize()
    refx = oracle.linear_bwd_input(S, c["dY"], NT)
    if gate:
        refx = refx * (H > 0)
    _assert_tol("fused dX", _np(dX), refx)
    _assert_tol("fused dW", _np(dW), oracle.linear_bwd_weight(S, c["X"], c["dY"], NT))
    # the separate dX kernel does the same products; the stream-K fused pass only
    # regroups the sums of items cut between CTAs (a + b): agreement to fp32 rounding
    dX2 = sp.sp_linear_bwd_input(Wg, _dev(c["dY"]), H=None if H is None else _dev(H))
    torch.cuda.synchronize()
    if B >= 128 and B % 4 == 0:
        a, b = _np(dX), _np(dX2)
        assert np.max(np.abs(a - b)) <= 1e-5 * max(float(np.max(np.abs(b))), 1e-30)


def test_random_small_shape_sweep(sp):
    """SPEC acceptance sweep (S620-S630): 200 seeded instances with
    (R, C, B) uniform in [1, 128]^3 at sparsity 0, 0.5, 0.9, 0.99 and
    all-but-one (a single kept weight); fwd, dX, dW and the fused backward
    against the oracle (B not a multiple of 4 takes the ragged paths)."""
    g = synth.rng(2302)
    kinds = [0.0, 0.5, 0.9, 0.99, "one"]
    for i in range(200):
        R, C, B = (int(v) for v in g.integers(1, 129, size=3))
        k = kinds[i % len(kinds)]
        if k == "one":
            mask = np.zeros((R, C), np.uint8)
            mask[int(g.integers(R)), int(g.integers(C))] = 1
        else:
            mask = (g.random((R, C)) >= k).astype(np.uint8)
        W = synth.normal(g, (R, C), 1.0 / C)
        X = synth.normal(g, (C, B), 1.0)
        dY = synth.normal(g, (R, B), 1.0)
        tag = f"sweep {i}: {R}x{C} B={B} {k}"
        check_linear(sp, W, mask, X, dY, tag)
        S = oracle.csr_from_mask(W, mask)
        Wg = sp.sp_weight_create(_dev(W), _dev(mask))
        fdX, fdW = sp.sp_linear_bwd(Wg, _dev(X), _dev(dY))
        torch.cuda.synchronize()
        _assert_tol(f"{tag} fused dX", _np(fdX), oracle.linear_bwd_input(S, dY, NT))
        _assert_tol(f"{tag} fused dW", _np(fdW), oracle.linear_bwd_weight(S, X, dY, NT))


@pytest.mark.parametrize("R,C,B", [(768, 3072, 2048), (3072, 768, 16384), (500, 300, 200)])
def test_fused_backward_gate_is_x(sp, R, C, B):
    """The DP step's ReLU' gate is the layer input itself (H == X): the fused
    backward then reads the gate from the X rows it already holds in TMEM."""
    c = synth.linear_case(R, C, B, 0.05, 1.0 / C, R + 7 * B)
    X = np.maximum(c["X"], 0.0).astype(np.float32)   # a post-ReLU input (exact zeros)
    S = oracle.csr_from_mask(c["W"], c["mask"])
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    Xg = _dev(X)
    dX, dW = sp.sp_linear_bwd(Wg, Xg, _dev(c["dY"]), H=Xg)
    torch.cuda.synchronize()
    _assert_tol("fused dX (gate = X)", _np(dX), oracle.linear_bwd_input(S, c["dY"], NT) * (X > 0))
    _assert_tol("fused dW (gate = X)", _np(dW), oracle.linear_bwd_weight(S, X, c["dY"], NT))


@pytest.mark.parametrize("R,C,B,kind", [(3072, 768, 2052, "uniform"), (2048, 1536, 2308, "zipf"),
                                        (3000, 1000, 2560, "uniform")])
def test_split_source_spmm_shapes(sp, R, C, B, kind):
    """Shapes that take the default split-source SpMM (32-warp per-item grid,
    TMEM-mirrored tile rows) with a partial last batch slice, ragged row / column
    blocks (R, C not multiples of 128 / 192) and skewed rows."""
    c = synth.linear_case(R, C, B, 0.05, 1.0 / C, R + B, kind)
    check_linear(sp, c["W"], c["mask"], c["X"], c["dY"], f"split-source {R}x{C} B={B} {kind}")


# ---------------------------------------------------------------- conv, NCHW (SparseConvOverON)
@pytest.mark.parametrize("B,IC,OC,H,W,K,pad,d", [
    (4, 64, 48, 56, 56, 1, 0, 0.1),     # 1 x 1 on a large spatial input: the direct NCHW path (P397)
    (3, 16, 24, 28, 20, 1, 0, 0.2),     # 1 x 1, partial spatial tiles (nq x np tiles of 28 x 20)
    (1, 4, 4, 8, 8, 1, 0, 0.5),         # 1 x 1, one image
    (4, 32, 48, 56, 56, 3, 1, 0.1),     # 3 x 3 (column shifts of one float): permuted CHWN kernels
    (2, 16, 16, 28, 20, 5, 2, 0.2),     # K = 5
    (8, 16, 16, 14, 14, 3, 1, 0.2),     # W = 14 (not % 4)
])
def test_conv_nchw(sp, B, IC, OC, H, W, K, pad, d):
    """The NCHW entry points against the oracle's native NCHW conv (Eq. 3-5)."""
    c = synth.conv_case(OC=OC, IC=IC, H=H, W=W, KH=K, KW=K, pad=pad, B=B, density=d,
                        wvar=1.0 / (IC * K * K), seed=B * 11 + IC + OC + H + K)
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(c["mask"]))
    g = sp.conv_geom(Wg, B, H, W, pad)
    Xn, dOn = oracle.chwn_to_nchw(c["X"]), oracle.chwn_to_nchw(c["dY"])
    X, dY = _dev(Xn), _dev(dOn)
    Y = sp.sp_conv2d_fwd_nchw(Wg, g, X)
    pf = sp.last_path()
    dX = sp.sp_conv2d_bwd_input_nchw(Wg, g, dY)
    dW = sp.sp_conv2d_bwd_weight_nchw(Wg, g, X, dY)
    fdX, fdW = sp.sp_conv2d_bwd_nchw(Wg, g, X, dY)
    pb = sp.last_path()
    torch.cuda.synchronize()
    F = oracle.conv_format(c["W"], c["mask"])
    tag = f"nchw B={B} {IC}->{OC} {H}x{W} K={K} pad={pad} [{pf} / {pb}]"
    _assert_tol(f"{tag} Y", _np(Y), oracle.conv2d_fwd(F, Xn, pad, NT))
    rdX, rdW = oracle.conv2d_bwd(F, Xn, dOn, pad)
    _assert_tol(f"{tag} dX", _np(dX), rdX)
    _assert_tol(f"{tag} dW", _np(dW), rdW)
    _assert_tol(f"{tag} fused dX", _np(fdX), rdX)
    _assert_tol(f"{tag} fused dW", _np(fdW), rdW)
    if K == 1 and pad == 0 and W % 4 == 0:
        assert "permute" not in pf and "permute" not in pb, (pf, pb)


@pytest.mark.parametrize("B", [256, 2048, 90])
def test_split_rows_dense_head(sp, B):
    """Rows far longer than the mean (Zipf heads) are dealt into part rows in
    the forward tilings and summed by split_rows_reduce: fwd, fwd+ReLU and
    every backward product against the oracle, with a few fully dense rows."""
    R, C = 2048, 1536
    c = synth.linear_case(R, C, B, 0.03, 1.0 / C, 4321 + B)
    mask = c["mask"].copy()
    mask[[3, 700, 701, 2047], :] = 1          # dense head rows
    mask[1000, : C // 2] = 1                  # a half-dense row
    S = oracle.csr_from_mask(c["W"], mask)
    Wg = sp.sp_weight_create(_dev(c["W"]), _dev(mask))
    X, dY = _dev(c["X"]), _dev(c["dY"])
    Y = sp.sp_linear_fwd(Wg, X)
    p0 = sp.last_path()
    Yr = sp.sp_linear_fwd(Wg, X, relu=True)
    dX, dW = sp.sp_linear_bwd(Wg, X, dY)
    dW2 = sp.sp_linear_bwd_weight(Wg, X, dY)
    torch.cuda.synchronize()
    ref = oracle.linear_fwd(S, c["X"], NT)
    _assert_tol(f"split fwd B={B} [{p0}]", _np(Y), ref)
    _assert_tol(f"split fwd relu B={B}", _np(Yr), np.maximum(ref, 0.0))
    _assert_tol(f"split dX B={B}", _np(dX), oracle.linear_bwd_input(S, c["dY"], NT))
    refw = oracle.linear_bwd_weight(S, c["X"], c["dY"], NT)
    _assert_tol(f"split dW B={B}", _np(dW), refw)
    _assert_tol(f"split dW alone B={B}", _np(dW2), refw)
    if B % 4 == 0:
        assert "split_rows_reduce" in p0.split("+") or "spmm_gather" in p0, p0

"""Pins of the oracle against things other than itself (CPU only).

Each test names the passage or the mathematical fact it pins, and is chosen so
that a plausible mistake in oracle/ (a dropped term, a wrong sign or index, a
transposed operand, a wrong CSC/perm mapping) fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))


def _layer(R, C, B, d, seed):
    g = synth.rng(seed)
    mask = synth.bernoulli_mask(g, R, C, d)
    W = synth.normal(g, (R, C), 1.0 / C)
    X = synth.normal(g, (C, B), 1.0)
    G = synth.normal(g, (R, B), 1.0)
    return W, mask, X, G


# --------------------------------------------------------------------------
# CSR / CSC / perm structure (P153-P154, P183) -- brute-force mask scans
# --------------------------------------------------------------------------
@pytest.mark.parametrize("R,C,d,seed", [(1, 1, 1.0, 0), (7, 5, 0.5, 1), (64, 48, 0.15, 2),
                                        (33, 70, 0.02, 3), (16, 16, 0.0, 4), (9, 13, 1.0, 5)])
def test_csr_csc_structure_bruteforce(R, C, d, seed):
    W, mask, _, _ = _layer(R, C, 2, d, seed)
    S = oracle.csr_from_mask(W, mask)
    rows, cols = np.nonzero(mask)                    # row-major scan == CSR order
    assert S.nnz == len(rows)
    assert np.array_equal(S.row_ptr, np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=R))]))
    assert np.array_equal(S.col_idx, cols)
    assert np.array_equal(S.vals, W[rows, cols].astype(np.float64))
    # CSC: column-major scan of the mask
    ccols, crows = np.nonzero(mask.T)
    assert np.array_equal(S.col_ptr, np.concatenate([[0], np.cumsum(np.bincount(ccols, minlength=C))]))
    assert np.array_equal(S.row_idx, crows)
    # perm is a bijection onto CSR slots and points at the same (r, c)
    assert np.array_equal(np.sort(S.perm), np.arange(S.nnz))
    assert np.array_equal(rows[S.perm], crows)
    assert np.array_equal(cols[S.perm], ccols)


def test_csr_spec_examples():
    # SPEC S120-S121 [TRIVIAL]: 2x2 identity -> row_ptr [0,1,2]; all-zero -> empty
    S = oracle.csr_from_mask(np.eye(2), np.eye(2, dtype=np.uint8))
    assert S.row_ptr.tolist() == [0, 1, 2] and S.col_idx.tolist() == [0, 1]
    assert S.vals.tolist() == [1.0, 1.0]
    Z = oracle.csr_from_mask(np.ones((2, 2)), np.zeros((2, 2), np.uint8))
    assert Z.row_ptr.tolist() == [0, 0, 0] and Z.nnz == 0


def test_structure_comes_from_mask_not_values():
    # on-mask zeros are stored, off-mask values ignored
    dense = np.array([[0.0, 5.0], [7.0, 0.0]])
    mask = np.array([[1, 0], [1, 1]], np.uint8)
    S = oracle.csr_from_mask(dense, mask)
    assert S.row_ptr.tolist() == [0, 1, 3]
    assert S.col_idx.tolist() == [0, 0, 1]
    assert S.vals.tolist() == [0.0, 7.0, 0.0]


# --------------------------------------------------------------------------
# Linear forward (P141): masked-dense library matmul, special cases
# --------------------------------------------------------------------------
@pytest.mark.parametrize("R,C,B,d,seed", [(64, 48, 33, 0.15, 10), (40, 90, 7, 0.05, 11),
                                          (5, 3, 1, 1.0, 12), (128, 96, 64, 0.02, 13)])
def test_fwd_vs_masked_dense(R, C, B, d, seed):
    W, mask, X, _ = _layer(R, C, B, d, seed)
    S = oracle.csr_from_mask(W, mask)
    Y = oracle.linear_fwd(S, X)
    ref = (W.astype(np.float64) * mask) @ X.astype(np.float64)
    np.testing.assert_allclose(Y, ref, rtol=1e-12, atol=1e-12)


def test_fwd_special_cases():
    X = synth.normal(synth.rng(3), (6, 5), 1.0)
    S = oracle.csr_from_mask(np.eye(6), np.eye(6, dtype=np.uint8))
    assert np.array_equal(oracle.linear_fwd(S, X), X.astype(np.float64))   # identity (S292)
    Z = oracle.csr_from_mask(np.ones((4, 6)), np.zeros((4, 6), np.uint8))
    assert np.array_equal(oracle.linear_fwd(Z, X), np.zeros((4, 5)))     # empty (S291)


# --------------------------------------------------------------------------
# Input gradient (Eq. 1, P143-P145)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("R,C,B,d,seed", [(64, 48, 33, 0.15, 20), (17, 80, 5, 0.1, 21)])
def test_dx_adjoint_and_masked_dense(R, C, B, d, seed):
    W, mask, X, G = _layer(R, C, B, d, seed)
    S = oracle.csr_from_mask(W, mask)
    dX = oracle.linear_bwd_input(S, G)
    # masked-dense library reference W^T G
    ref = (W.astype(np.float64) * mask).T @ G.astype(np.float64)
    np.testing.assert_allclose(dX, ref, rtol=1e-12, atol=1e-12)
    # adjoint identity <W X, G> = <X, W^T G> (closed form)
    lhs = float(np.sum(oracle.linear_fwd(S, X) * G))
    rhs = float(np.sum(X.astype(np.float64) * dX))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_dx_finite_difference():
    # L(X) = <G, W X> is linear in X, so central FD is exact up to rounding
    W, mask, X, G = _layer(9, 7, 3, 0.4, 22)
    S = oracle.csr_from_mask(W, mask)
    dX = oracle.linear_bwd_input(S, G)
    X64 = X.astype(np.float64)
    eps = 1e-3
    for c in range(7):
        for b in range(3):
            Xp, Xm = X64.copy(), X64.copy()
            Xp[c, b] += eps
            Xm[c, b] -= eps
            fd = (np.sum(G * oracle.linear_fwd(S, Xp)) - np.sum(G * oracle.linear_fwd(S, Xm))) / (2 * eps)
            assert abs(fd - dX[c, b]) < 1e-9


# --------------------------------------------------------------------------
# Weight gradient (Eq. 2, P146-P148, SDDMM P151)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("R,C,B,d,seed", [(64, 48, 33, 0.15, 30), (20, 31, 129, 0.2, 31)])
def test_dw_gather_and_closed_form(R, C, B, d, seed):
    W, mask, X, G = _layer(R, C, B, d, seed)
    S = oracle.csr_from_mask(W, mask)
    dW = oracle.linear_bwd_weight(S, X, G)
    full = G.astype(np.float64) @ X.astype(np.float64).T           # dense dY X^T
    rows, cols = np.nonzero(mask)
    np.testing.assert_allclose(dW, full[rows, cols], rtol=1e-12, atol=1e-12)
    # sum_j dW_j V_j = <G, V X> for any V supported on the mask
    V = synth.normal(synth.rng(seed + 100), (R, C), 1.0).astype(np.float64) * mask
    lhs = float(np.sum(dW * V[rows, cols]))
    rhs = float(np.sum(G * (V @ X.astype(np.float64))))
    assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(rhs))
    # densify: exactly +0.0 off the mask (north star)
    D = oracle.densify(S, dW)
    off = D[mask == 0]
    assert np.all(off == 0.0) and not np.any(np.signbit(off))
    assert np.array_equal(D[rows, cols], dW)


def test_dw_finite_difference():
    W, mask, X, G = _layer(6, 8, 4, 0.5, 32)
    S = oracle.csr_from_mask(W, mask)
    dW = oracle.linear_bwd_weight(S, X, G)
    eps = 1e-3
    for j in range(S.nnz):
        vp, vm = S.vals.copy(), S.vals.copy()
        vp[j] += eps
        vm[j] -= eps
        fd = (np.sum(G * oracle.linear_fwd(S.with_vals(vp), X))
              - np.sum(G * oracle.linear_fwd(S.with_vals(vm), X))) / (2 * eps)
        assert abs(fd - dW[j]) < 1e-9


def test_identity_mask_dw():
    # SPEC S301 [TRIVIAL]: identity mask -> dW_j = <dY row j, X row j>
    g = synth.rng(33)
    X = synth.normal(g, (5, 11), 1.0)
    G = synth.normal(g, (5, 11), 1.0)
    S = oracle.csr_from_mask(np.eye(5), np.eye(5, dtype=np.uint8))
    dW = oracle.linear_bwd_weight(S, X, G)
    np.testing.assert_allclose(dW, np.sum(X.astype(np.float64) * G, axis=1), rtol=1e-14)


def test_thread_count_invariance_bitwise():
    W, mask, X, G = _layer(130, 70, 19, 0.1, 40)
    S = oracle.csr_from_mask(W, mask)
    for f in (lambda n: oracle.linear_fwd(S, X, n), lambda n: oracle.linear_bwd_input(S, G, n),
              lambda n: oracle.linear_bwd_weight(S, X, G, n)):
        assert np.array_equal(f(1), f(4))


# --------------------------------------------------------------------------
# Convolution (Eqs. 3-5, Alg. 2, the 4-array format)
# --------------------------------------------------------------------------
def test_conv_format_paper_worked_example():
    with open(os.path.join(HERE, "golden", "conv_format_example.json")) as f:
        ex = json.load(f)
    shape = tuple(ex["shape"])
    dense = np.zeros(shape)
    mask = np.zeros(shape, np.uint8)
    for k, (oc, ic, x, y) in ex["entries"].items():
        dense[oc, ic, x, y] = ex["values"][k]
        mask[oc, ic, x, y] = 1
    F = oracle.conv_format(dense, mask)
    assert F.och.tolist() == ex["W_och"]
    assert F.ich.tolist() == ex["W_ich"]
    assert F.wx.tolist() == ex["W_x"]
    assert F.wy.tolist() == ex["W_y"]
    assert F.vals.tolist() == ex["W_vals_reading_C8"]


def _conv(B, IC, OC, H, W, K, pad, d, seed):
    c = synth.conv_case(OC=OC, IC=IC, H=H, W=W, KH=K, KW=K, pad=pad, B=B, density=d,
                        wvar=1.0 / (IC * K * K), seed=seed)
    return c


@pytest.mark.parametrize("B,IC,OC,H,W,K,pad,d,seed", [
    (2, 3, 4, 7, 7, 3, 1, 0.5, 50),      # SPEC S347-style geometry
    (3, 6, 5, 9, 9, 3, 1, 0.1, 51),
    (2, 4, 3, 6, 5, 3, 0, 0.4, 52),
    (1, 2, 2, 5, 5, 5, 2, 0.6, 53),
    (2, 3, 2, 4, 6, 1, 0, 0.7, 54),
])
def test_conv_vs_torch_float64(B, IC, OC, H, W, K, pad, d, seed):
    torch = pytest.importorskip("torch")
    c = _conv(B, IC, OC, H, W, K, pad, d, seed)
    F = oracle.conv_format(c["W"], c["mask"])
    X = oracle.chwn_to_nchw(c["X"])
    dO = oracle.chwn_to_nchw(c["dY"])
    Wm = torch.tensor(c["W"].astype(np.float64) * c["mask"], requires_grad=True)
    Xt = torch.tensor(X.astype(np.float64), requires_grad=True)
    Ot = torch.nn.functional.conv2d(Xt, Wm, padding=pad)
    Ot.backward(torch.tensor(dO.astype(np.float64)))
    O = oracle.conv2d_fwd(F, X, pad)
    np.testing.assert_allclose(O, Ot.detach().numpy(), rtol=1e-12, atol=1e-12)
    dX, dW = oracle.conv2d_bwd(F, X, dO, pad)
    np.testing.assert_allclose(dX, Xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    sel = np.nonzero(c["mask"])        # lexicographic (oc, ic, x, y) == storage order
    np.testing.assert_allclose(dW, Wm.grad.numpy()[sel], rtol=1e-12, atol=1e-12)


def test_conv_k1_reduces_to_linear():
    # SPEC S229/S346: K=1, pad=0 is a linear layer over channels per pixel
    c = _conv(3, 5, 4, 4, 3, 1, 0, 0.5, 55)
    F = oracle.conv_format(c["W"], c["mask"])
    X = oracle.chwn_to_nchw(c["X"])
    dO = oracle.chwn_to_nchw(c["dY"])
    O = oracle.conv2d_fwd(F, X, 0)
    S = oracle.csr_from_mask(c["W"][:, :, 0, 0], c["mask"][:, :, 0, 0])
    Xl = c["X"].reshape(5, -1)                        # [IC][(H W B)]
    Yl = oracle.linear_fwd(S, Xl)
    np.testing.assert_allclose(oracle.nchw_to_chwn(O).reshape(4, -1), Yl, rtol=1e-13, atol=1e-13)
    dX, dW = oracle.conv2d_bwd(F, X, dO, 0)
    np.testing.assert_allclose(oracle.nchw_to_chwn(dX).reshape(5, -1),
                               oracle.linear_bwd_input(S, c["dY"].reshape(4, -1)), rtol=1e-13,
                               atol=1e-13)
    np.testing.assert_allclose(dW, oracle.linear_bwd_weight(S, Xl, c["dY"].reshape(4, -1)),
                               rtol=1e-13, atol=1e-13)


def test_conv_full_kernel_reduces_to_linear():
    # SPEC S253: K = H = W, pad 0 -> linear over the flattened input
    c = _conv(4, 3, 5, 3, 3, 3, 0, 0.5, 56)
    F = oracle.conv_format(c["W"], c["mask"])
    X = oracle.chwn_to_nchw(c["X"])
    O = oracle.conv2d_fwd(F, X, 0)                    # [B][OC][1][1]
    S = oracle.csr_from_mask(c["W"].reshape(5, -1), c["mask"].reshape(5, -1))
    Yl = oracle.linear_fwd(S, c["X"].reshape(27, -1))  # CHW flattened == (ic, x, y)
    np.testing.assert_allclose(O[:, :, 0, 0].T, Yl, rtol=1e-13, atol=1e-13)


def test_conv_finite_difference_tiny():
    c = _conv(2, 2, 2, 4, 4, 3, 1, 0.6, 57)
    F = oracle.conv_format(c["W"], c["mask"])
    X = oracle.chwn_to_nchw(c["X"]).astype(np.float64)
    G = oracle.chwn_to_nchw(c["dY"]).astype(np.float64)
    dX, dW = oracle.conv2d_bwd(F, X, G, 1)
    eps = 1e-3
    L = lambda FF, XX: float(np.sum(G * oracle.conv2d_fwd(FF, XX, 1)))
    for idx in [(0, 0, 0, 0), (1, 1, 3, 2), (0, 1, 2, 3), (1, 0, 1, 1)]:
        Xp, Xm = X.copy(), X.copy()
        Xp[idx] += eps
        Xm[idx] -= eps
        assert abs((L(F, Xp) - L(F, Xm)) / (2 * eps) - dX[idx]) < 1e-9
    for j in range(F.nnz):
        vp, vm = F.vals.copy(), F.vals.copy()
        vp[j] += eps
        vm[j] -= eps
        Fp = oracle.ConvFormat(F.OC, F.IC, F.KH, F.KW, F.och, F.ich, F.wx, F.wy, vp)
        Fm = oracle.ConvFormat(F.OC, F.IC, F.KH, F.KW, F.och, F.ich, F.wx, F.wy, vm)
        assert abs((L(Fp, X) - L(Fm, X)) / (2 * eps) - dW[j]) < 1e-9


# --------------------------------------------------------------------------
# cfg5 MLP composition (north star; C18 loss, C26 ReLU')
# --------------------------------------------------------------------------
def _tiny_mlp(seed=60, T=6):
    c = synth.mlp_case(blocks=2, d_model=6, d_ff=10, T=T, density=0.5, seed=seed)
    layers = [(oracle.csr_from_mask(w1, m1), oracle.csr_from_mask(w2, m2))
              for (w1, m1, w2, m2) in c["layers"]]
    return c, layers


def test_mlp_finite_difference():
    c, layers = _tiny_mlp()
    out = oracle.mlp_step(layers, c["X0"], c["target"])
    eps = 1e-6
    for l in range(2):
        for which in range(2):
            S = layers[l][which]
            for j in range(0, S.nnz, 3):
                vp, vm = S.vals.copy(), S.vals.copy()
                vp[j] += eps
                vm[j] -= eps
                lp = [list(p) for p in layers]
                lp[l][which] = S.with_vals(vp)
                lm = [list(p) for p in layers]
                lm[l][which] = S.with_vals(vm)
                fd = (oracle.mlp_step(lp, c["X0"], c["target"])["loss"]
                      - oracle.mlp_step(lm, c["X0"], c["target"])["loss"]) / (2 * eps)
                assert abs(fd - out["dW"][l][which][j]) < 1e-5 * max(1.0, abs(fd))
    # loss is 1/2 sum (Y - T)^2 (C18)
    d = out["Y"] - c["target"].astype(np.float64)
    assert out["loss"] == pytest.approx(0.5 * float(np.sum(d * d)), rel=1e-14)


def test_mlp_dp_algebra():
    # sum over token shards of per-shard dW == full-batch dW
    c, layers = _tiny_mlp(61, T=10)
    full = oracle.mlp_step(layers, c["X0"], c["target"])
    for G in (2, 3):
        acc = None
        for r in range(G):
            lo, hi = synth.token_shard(10, G, r)
            o = oracle.mlp_step(layers, c["X0"][:, lo:hi], c["target"][:, lo:hi])
            flat = np.concatenate([np.concatenate(p) for p in o["dW"]])
            acc = flat if acc is None else acc + flat
        ref = np.concatenate([np.concatenate(p) for p in full["dW"]])
        np.testing.assert_allclose(acc, ref, rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------------
# Synthetic generator structure (C14) -- parity unpinned vs the paper
# --------------------------------------------------------------------------
@pytest.mark.parametrize("d", [0.2, 0.05, 0.01])
def test_zipf_counts_structure(d):
    n1 = synth.zipf_row_counts(synth.rng(7), 512, 512, d)
    n2 = synth.zipf_row_counts(synth.rng(7), 512, 512, d)
    assert np.array_equal(n1, n2)
    assert n1.sum() == int(round(d * 512 * 512))
    assert n1.min() >= 0 and n1.max() <= 512
    assert n1.max() > 4 * np.median(n1)      # skewed


def test_token_shard_partition():
    for T, G in [(16384, 8), (10, 3), (7, 4)]:
        rs = [synth.token_shard(T, G, r) for r in range(G)]
        assert rs[0][0] == 0 and rs[-1][1] == T
        assert all(rs[i][1] == rs[i + 1][0] for i in range(G - 1))

"""cfg5 data-parallel MLP step on the GPU vs the oracle (SURVEY §8(c) C19:
layer-local parity -- the oracle recomputes every layer from the GPU's own
saved inputs -- plus end-to-end loss agreement and the ReLU-flip count)."""
import numpy as np
import pytest

import oracle
import synth
from conftest import tol_ok

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
NT = min(8, oracle.threads_available())


def _np(t):
    return t.detach().cpu().numpy()


def _ok(name, got, ref):
    ok, err, bound = tol_ok(got, ref)
    assert ok, f"{name}: max|err| {err:.3e} > {bound:.3e}"


@pytest.mark.parametrize("fused", [True, False])
def test_mlp_step_layer_local_parity(fused):
    from paper_2302_04852_b200.dp import SparseMLP
    T = 1024
    c = synth.mlp_case(blocks=12, d_model=768, d_ff=3072, T=T, density=0.05, seed=5)
    m = SparseMLP(c["layers"], T, "cuda", fused=fused)
    m.set_batch(torch.from_numpy(c["X0"]), torch.from_numpy(c["target"]), non_blocking=False)
    loss = float(m.forward())
    trace = []
    m.backward(allreduce=False, trace=trace)
    torch.cuda.synchronize()
    S = [(oracle.csr_from_mask(w1, m1), oracle.csr_from_mask(w2, m2)) for (w1, m1, w2, m2) in c["layers"]]
    # forward, layer-local
    for l, (S1, S2) in enumerate(S):
        X = _np(m.X[l])
        H = _np(m.H[l])
        _ok(f"H[{l}]", H, np.maximum(oracle.linear_fwd(S1, X, NT), 0.0))
        _ok(f"X[{l + 1}]", _np(m.X[l + 1]), oracle.linear_fwd(S2, H, NT))
    Y = _np(m.X[12]).astype(np.float64)
    d = Y - c["target"]
    assert loss == pytest.approx(0.5 * float(np.sum(d * d)), rel=1e-5)
    # backward, layer-local from the GPU's own dY_in of each block
    for (l, dY_in, dZ, dX_out) in trace:
        S1, S2 = S[l]
        X, H, dYl = _np(m.X[l]), _np(m.H[l]), _np(dY_in)
        refZ = oracle.linear_bwd_input(S2, dYl, NT) * (H > 0)
        _ok(f"dZ[{l}]", _np(dZ), refZ)
        dW1, dW2 = m.dW[l]
        _ok(f"dW2[{l}]", _np(dW2), oracle.linear_bwd_weight(S2, H, dYl, NT))
        _ok(f"dW1[{l}]", _np(dW1), oracle.linear_bwd_weight(S1, X, _np(dZ), NT))
        _ok(f"dX[{l}]", _np(dX_out), oracle.linear_bwd_input(S1, _np(dZ), NT))
    # end to end against the oracle's own full forward: loss and flip count
    ref = oracle.mlp_step(S, c["X0"], c["target"], NT)
    assert loss == pytest.approx(ref["loss"], rel=1e-4)
    flips = sum(int(np.sum((_np(m.H[l]) > 0) != (ref["acts"][l][1] > 0))) for l in range(12))
    assert flips < 1e-4 * 12 * 3072 * T, flips


def test_mlp_sgd_updates_only_kept_weights():
    from paper_2302_04852_b200.dp import SparseMLP
    c = synth.mlp_case(blocks=2, d_model=768, d_ff=3072, T=256, density=0.05, seed=6)
    m = SparseMLP(c["layers"], 256, "cuda")
    m.set_batch(torch.from_numpy(c["X0"]), torch.from_numpy(c["target"]), non_blocking=False)
    before = [(W1.vals.clone(), W2.vals.clone()) for W1, W2 in m.W]
    m.step(1e-3)
    torch.cuda.synchronize()
    for l, ((W1, W2), (b1, b2), (d1, d2)) in enumerate(zip(m.W, before, m.dW)):
        np.testing.assert_allclose(_np(W1.vals), _np(b1) - 1e-3 * _np(d1), rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(_np(W2.vals), _np(b2) - 1e-3 * _np(d2), rtol=1e-6, atol=1e-7)
        # dW densifies to exact zeros off each layer's mask
        for Wh, dd, mask in ((W1, d1, c["layers"][l][1]), (W2, d2, c["layers"][l][3])):
            D = _np(Wh.to_dense(dd))
            assert np.all(D[mask == 0] == 0.0)


def test_mlp_full_size_sampled():
    """cfg5 at its full size in bench.py's launch configuration (16384 tokens on
    one GPU, fused backward): layer-local parity on 64 sampled token columns
    for the forward and dX products (columns are independent), and on every
    nonzero for the dW of the first and last blocks (full batch)."""
    from paper_2302_04852_b200.dp import SparseMLP
    T = 16384
    c = synth.mlp_case(blocks=12, d_model=768, d_ff=3072, T=T, density=0.05, seed=5)
    m = SparseMLP(c["layers"], T, "cuda")
    m.set_batch(torch.from_numpy(c["X0"]), torch.from_numpy(c["target"]), non_blocking=False)
    m.forward()
    trace = []
    m.backward(allreduce=False, trace=trace)
    torch.cuda.synchronize()
    cols = np.sort(synth.rng(55).choice(T, 64, replace=False))
    S = [(oracle.csr_from_mask(w1, m1), oracle.csr_from_mask(w2, m2)) for (w1, m1, w2, m2) in c["layers"]]
    for l in (0, 5, 11):
        S1, S2 = S[l]
        X = np.ascontiguousarray(_np(m.X[l])[:, cols])
        H = np.ascontiguousarray(_np(m.H[l])[:, cols])
        _ok(f"H[{l}] sampled", H, np.maximum(oracle.linear_fwd(S1, X, NT), 0.0))
        _ok(f"X[{l + 1}] sampled", _np(m.X[l + 1])[:, cols], oracle.linear_fwd(S2, H, NT))
    for (l, dY_in, dZ, dX_out) in trace:
        if l not in (0, 11):
            continue
        S1, S2 = S[l]
        Hs = _np(m.H[l])[:, cols]
        dYs = np.ascontiguousarray(_np(dY_in)[:, cols])
        dZs = np.ascontiguousarray(_np(dZ)[:, cols])
        _ok(f"dZ[{l}] sampled", dZs, oracle.linear_bwd_input(S2, dYs, NT) * (Hs > 0))
        _ok(f"dX[{l}] sampled", _np(dX_out)[:, cols], oracle.linear_bwd_input(S1, dZs, NT))
        dW1, dW2 = m.dW[l]
        _ok(f"dW2[{l}] full batch", _np(dW2), oracle.linear_bwd_weight(S2, _np(m.H[l]), _np(dY_in), NT))
        _ok(f"dW1[{l}] full batch", _np(dW1), oracle.linear_bwd_weight(S1, _np(m.X[l]), _np(dZ), NT))


def test_mlp_sharded_step_matches_full_batch():
    """The data-parallel algebra on the GPU path without a collective (SURVEY
    §4 "simulated ranks"): G token shards run one after another on one GPU;
    their forward outputs are the full-batch outputs of their columns and the
    sum of their dW is the full-batch dW (what all_reduce(SUM) computes)."""
    from paper_2302_04852_b200.dp import SparseMLP
    T, G = 4096, 4
    c = synth.mlp_case(blocks=2, d_model=768, d_ff=3072, T=T, density=0.05, seed=8)
    full = SparseMLP(c["layers"], T, "cuda")
    full.set_batch(torch.from_numpy(c["X0"]), torch.from_numpy(c["target"]), non_blocking=False)
    full.forward()
    full.backward(allreduce=False)
    dW_sum = torch.zeros_like(full.dW_flat)
    for g in range(G):
        lo, hi = synth.token_shard(T, G, g)
        m = SparseMLP(c["layers"], hi - lo, "cuda")
        m.set_batch(torch.from_numpy(np.ascontiguousarray(c["X0"][:, lo:hi])),
                    torch.from_numpy(np.ascontiguousarray(c["target"][:, lo:hi])), non_blocking=False)
        m.forward()
        m.backward(allreduce=False)
        _ok(f"shard {g} output", _np(m.X[2]), _np(full.X[2])[:, lo:hi])
        dW_sum += m.dW_flat
    torch.cuda.synchronize()
    _ok("sum of shard dW", _np(dW_sum), _np(full.dW_flat))


def test_managed_weights_stay_in_sync():
    """sp_weight_sgd on a managed handle (products skip the per-launch refresh
    of the tiled weights) gives bitwise the results of sp_sgd + refreshing
    products on an unmanaged handle, over several steps and every kernel that
    reads tiled weights; sp_weight_set_managed after an external vals write
    makes the next products pick it up."""
    from paper_2302_04852_b200 import sparseprop as sp
    c = synth.linear_case(3072, 768, 2048, 0.05, 1.0 / 768, 91)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    Wm = sp.sp_weight_create(dev(c["W"]), dev(c["mask"]))
    Wu = sp.sp_weight_create(dev(c["W"]), dev(c["mask"]))
    sp.sp_weight_set_managed(Wm, True)
    X, dY = dev(c["X"]), dev(c["dY"])
    g = torch.Generator(device="cuda").manual_seed(3)
    for step in range(3):
        dW = torch.randn(Wm.nnz, device="cuda", generator=g)
        sp.sp_weight_sgd(Wm, dW, 1e-2)
        sp.sp_sgd(Wu.vals, dW, 1e-2)
        for f in (lambda W: sp.sp_linear_fwd(W, X), lambda W: sp.sp_linear_fwd(W, X, relu=True),
                  lambda W: sp.sp_linear_bwd_input(W, dY), lambda W: sp.sp_linear_bwd(W, X, dY)[0]):
            assert torch.equal(f(Wm), f(Wu)), step
    assert torch.equal(Wm.vals, Wu.vals)
    # an external write while managed is picked up after sp_weight_set_managed
    Wm.vals.mul_(0.5)
    Wu.vals.mul_(0.5)
    sp.sp_weight_set_managed(Wm, True)
    assert torch.equal(sp.sp_linear_fwd(Wm, X), sp.sp_linear_fwd(Wu, X))
    torch.cuda.synchronize()
    S = oracle.csr_from_mask(c["W"], c["mask"]).with_vals(_np(Wm.vals))
    _ok("managed fwd vs oracle", _np(sp.sp_linear_fwd(Wm, X)), oracle.linear_fwd(S, c["X"], NT))


def test_mlp_two_steps_then_forward_matches_oracle():
    """Training state stays coherent across steps (managed handles): after two
    SGD steps the next forward is layer-local equal to the oracle's with the
    updated weights."""
    from paper_2302_04852_b200.dp import SparseMLP
    T = 512
    c = synth.mlp_case(blocks=2, d_model=768, d_ff=3072, T=T, density=0.05, seed=12)
    m = SparseMLP(c["layers"], T, "cuda")
    m.set_batch(torch.from_numpy(c["X0"]), torch.from_numpy(c["target"]), non_blocking=False)
    m.step(1e-3)
    m.step(1e-3)
    m.forward()
    torch.cuda.synchronize()
    for l, ((w1, m1, w2, m2), (W1, W2)) in enumerate(zip(c["layers"], m.W)):
        S1 = oracle.csr_from_mask(w1, m1).with_vals(_np(W1.vals))
        S2 = oracle.csr_from_mask(w2, m2).with_vals(_np(W2.vals))
        X, H = _np(m.X[l]), _np(m.H[l])
        _ok(f"H[{l}] after 2 steps", H, np.maximum(oracle.linear_fwd(S1, X, NT), 0.0))
        _ok(f"X[{l + 1}] after 2 steps", _np(m.X[l + 1]), oracle.linear_fwd(S2, H, NT))


def test_graph_captured_step_matches_eager():
    """The whole step captured once in a CUDA graph (bench.py's timed loop) and
    replayed gives bitwise the eager steps' weights and loss: the same kernels
    with the same arguments, scratch from graph memory nodes."""
    from paper_2302_04852_b200.dp import SparseMLP
    T = 2048
    c = synth.mlp_case(blocks=3, d_model=768, d_ff=3072, T=T, density=0.05, seed=21)
    X0, Tg = torch.from_numpy(c["X0"]), torch.from_numpy(c["target"])
    a = SparseMLP(c["layers"], T, "cuda")
    b = SparseMLP(c["layers"], T, "cuda")
    for m in (a, b):
        m.set_batch(X0, Tg, non_blocking=False)
    for _ in range(3):
        la = a.step(1e-6)
    g = b.capture(1e-6)      # runs one eager (warm) step, then captures one
    g.replay()               # step 2
    g.replay()               # step 3
    torch.cuda.synchronize()
    assert torch.isfinite(la).all() and torch.equal(la, b.loss)
    for (A1, A2), (B1, B2) in zip(a.W, b.W):
        assert torch.equal(A1.vals, B1.vals) and torch.equal(A2.vals, B2.vals)
    assert torch.equal(a.dW_flat, b.dW_flat)


def test_batched_sgd_matches_per_handle():
    """sp_weights_sgd (one kernel for all of a model's handles) gives bitwise the
    vals and products of one sp_weight_sgd per handle, including the lazily
    refreshed tilings (a product after the update reads a tiling the step did
    not use)."""
    from paper_2302_04852_b200 import sparseprop as sp
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    cases = [synth.linear_case(3072, 768, 256, 0.05, 1.0 / 768, 61), synth.linear_case(768, 3072, 256, 0.05, 1.0 / 3072, 62),
             synth.linear_case(500, 300, 128, 0.1, 1.0 / 300, 63)]
    A = [sp.sp_weight_create(dev(c["W"]), dev(c["mask"])) for c in cases]
    Bh = [sp.sp_weight_create(dev(c["W"]), dev(c["mask"])) for c in cases]
    for W in A + Bh:
        sp.sp_weight_set_managed(W, True)
    g = torch.Generator(device="cuda").manual_seed(5)
    for step in range(3):
        for c, Wa, Wb in zip(cases, A, Bh):  # a product per handle (marks the tilings it reads)
            X = dev(c["X"])
            assert torch.equal(sp.sp_linear_fwd(Wa, X), sp.sp_linear_fwd(Wb, X)), step
        dWs = [torch.randn(W.nnz, device="cuda", generator=g) for W in A]
        sp.sp_weights_sgd(A, dWs, 1e-2)
        for Wb, d in zip(Bh, dWs):
            sp.sp_weight_sgd(Wb, d, 1e-2)
    for c, Wa, Wb in zip(cases, A, Bh):
        assert torch.equal(Wa.vals, Wb.vals)
        X, dY = dev(c["X"]), dev(c["dY"])
        for f in (lambda W: sp.sp_linear_fwd(W, X), lambda W: sp.sp_linear_bwd_input(W, dY),
                  lambda W: sp.sp_linear_bwd(W, X, dY)[0]):
            assert torch.equal(f(Wa), f(Wb))
    torch.cuda.synchronize()
    c = cases[0]
    S = oracle.csr_from_mask(c["W"], c["mask"]).with_vals(_np(A[0].vals))
    _ok("batched-SGD handle bwd_input vs oracle", _np(sp.sp_linear_bwd_input(A[0], dev(c["dY"]))),
        oracle.linear_bwd_input(S, c["dY"], NT))


def test_managed_conv_handle_refreshes_taps_per_version():
    """A managed conv handle refreshes its tap tilings once per vals version: the
    products after sp_weight_sgd (and after an external write + set_managed)
    match an unmanaged handle holding the same vals."""
    from paper_2302_04852_b200 import sparseprop as sp
    c = synth.conv_case(OC=48, IC=32, H=10, W=10, KH=3, KW=3, pad=1, B=8, density=0.2, wvar=2.0 / 288, seed=71)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    Wm = sp.sp_weight_create(dev(c["W"]), dev(c["mask"]))
    Wu = sp.sp_weight_create(dev(c["W"]), dev(c["mask"]))
    sp.sp_weight_set_managed(Wm, True)
    g = sp.conv_geom(Wm, c["B"], c["H"], c["Wd"], c["pad"])
    X, dY = dev(c["X"]), dev(c["dY"])
    gen = torch.Generator(device="cuda").manual_seed(9)
    for step in range(3):
        for f in (lambda W: sp.sp_conv2d_fwd(W, g, X), lambda W: sp.sp_conv2d_bwd_input(W, g, dY),
                  lambda W: sp.sp_conv2d_bwd(W, g, X, dY)[0]):
            assert torch.equal(f(Wm), f(Wu)), step
            assert torch.equal(f(Wm), f(Wu)), step  # (second call: no refresh on the managed handle)
        d = torch.randn(Wm.nnz, device="cuda", generator=gen)
        sp.sp_weight_sgd(Wm, d, 1e-2)
        sp.sp_sgd(Wu.vals, d, 1e-2)
    Wm.vals.mul_(0.5)
    Wu.vals.mul_(0.5)
    sp.sp_weight_set_managed(Wm, True)
    assert torch.equal(sp.sp_conv2d_fwd(Wm, g, X), sp.sp_conv2d_fwd(Wu, g, X))

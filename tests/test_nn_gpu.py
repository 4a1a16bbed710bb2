"""Drop-in modules (P358) against PyTorch float64 autograd on the masked dense
weight: outputs and gradients (input and kept weights) for the sparse path,
the dense path of the dispatcher, and the automatic choice."""
import numpy as np
import pytest

import synth
from conftest import tol_ok

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ok(name, got, ref):
    ok, err, bound = tol_ok(got.detach().cpu().double().numpy(), ref.detach().cpu().double().numpy())
    assert ok, f"{name}: {err:.3e} > {bound:.3e}"


@pytest.mark.parametrize("mode", ["sparse", "dense", "auto"])
@pytest.mark.parametrize("feature_major", [False, True])
def test_sparse_linear_module(mode, feature_major):
    from paper_2302_04852_b200.nn import SparseLinear
    c = synth.linear_case(384, 256, 192, 0.1, 1.0 / 256, 31)
    m = SparseLinear(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda(),
                     feature_major=feature_major, mode=mode)
    X = torch.from_numpy(c["X"] if feature_major else c["X"].T.copy()).cuda().requires_grad_(True)
    G = torch.from_numpy(c["dY"] if feature_major else c["dY"].T.copy()).cuda()
    y = m(X)
    y.backward(G)
    torch.cuda.synchronize()
    # float64 reference
    Wm = torch.from_numpy(c["W"].astype(np.float64) * c["mask"]).requires_grad_(True)
    Xr = X.detach().cpu().double().requires_grad_(True)
    yr = (Wm @ Xr) if feature_major else (Xr @ Wm.t())
    yr.backward(G.cpu().double())
    _ok("y", y, yr)
    _ok("dX", X.grad, Xr.grad)
    rows, cols = np.nonzero(c["mask"])
    _ok("dvals", m.vals.grad, Wm.grad[rows, cols])
    if mode != "auto":
        assert m.impl == mode


def test_sparse_linear_optimizer_updates_kept_weights_only():
    from paper_2302_04852_b200.nn import SparseLinear
    c = synth.linear_case(256, 128, 128, 0.05, 1.0 / 128, 32)
    m = SparseLinear(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda(), mode="sparse")
    opt = torch.optim.SGD(m.parameters(), lr=0.1)
    x = torch.from_numpy(c["X"].T.copy()).cuda()
    before = m.W.to_dense().cpu().numpy()
    m(x).pow(2).sum().backward()
    opt.step()
    after = m.W.to_dense().cpu().numpy()
    assert np.all(after[c["mask"] == 0] == 0.0)
    assert np.any(after[c["mask"] == 1] != before[c["mask"] == 1])


@pytest.mark.parametrize("mode", ["sparse", "dense"])
def test_sparse_conv_module(mode):
    from paper_2302_04852_b200.nn import SparseConv2d
    c = synth.conv_case(OC=24, IC=16, H=9, W=9, KH=3, KW=3, pad=1, B=8, density=0.15, wvar=1.0 / 144, seed=33)
    m = SparseConv2d(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda(), padding=1, mode=mode)
    Xn = torch.from_numpy(np.ascontiguousarray(np.transpose(c["X"], (3, 0, 1, 2)))).cuda().requires_grad_(True)
    Gn = torch.from_numpy(np.ascontiguousarray(np.transpose(c["dY"], (3, 0, 1, 2)))).cuda()
    y = m(Xn)
    y.backward(Gn)
    torch.cuda.synchronize()
    Wm = torch.from_numpy(c["W"].astype(np.float64) * c["mask"]).requires_grad_(True)
    Xr = Xn.detach().cpu().double().requires_grad_(True)
    yr = torch.nn.functional.conv2d(Xr, Wm, padding=1)
    yr.backward(Gn.cpu().double())
    _ok("y", y, yr)
    _ok("dX", Xn.grad, Xr.grad)
    _ok("dvals", m.vals.grad, Wm.grad[np.nonzero(c["mask"])])


def test_gmp_mask_update_rebuilds_and_stays_exact():
    """F4: prune a module from 80 % to 95 % by magnitude; the rebuilt structure
    matches a fresh handle built from the pruned weights, and the module still
    matches the float64 reference."""
    from paper_2302_04852_b200.nn import SparseLinear
    from paper_2302_04852_b200.prune import prune_modules
    c = synth.linear_case(512, 384, 256, 0.2, 1.0 / 384, 34)
    m = SparseLinear(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda(), mode="sparse")
    rep = prune_modules([m], 0.95)
    assert abs(rep["sparsity"][0] - 0.95) < 1.0 / (512 * 384) + 1e-9
    assert rep["rebuild_s"] >= 0.0
    Wd = m.W.to_dense().cpu().double()
    kept = (m.W.to_dense(torch.ones(m.W.nnz, device="cuda")) != 0).cpu().numpy()
    assert np.all(kept <= c["mask"].astype(bool))              # nested in the old mask
    x = torch.from_numpy(c["X"].T.copy()).cuda()
    y = m(x)
    _ok("y after pruning", y, x.cpu().double() @ Wd.t())


def test_optimizer_built_before_pruning_keeps_stepping():
    """an optimizer built before a GMP update must keep training the
    kept weights (the Parameter object survives set_mask), and the handle whose
    vals the Parameter views stays alive while the Parameter does."""
    import gc
    import weakref
    from paper_2302_04852_b200.nn import SparseLinear
    from paper_2302_04852_b200.prune import prune_modules
    c = synth.linear_case(256, 192, 128, 0.3, 1.0 / 192, 35)
    m = SparseLinear(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda(), mode="sparse")
    p_before = m.vals
    opt = torch.optim.SGD(m.parameters(), lr=0.1, momentum=0.9)
    x = torch.from_numpy(c["X"].T.copy()).cuda()
    m(x).square().sum().backward()
    opt.step()
    prune_modules([m], 0.9, optimizer=opt)
    assert m.vals is p_before and m.vals.numel() == m.W.nnz
    before = m.W.vals.clone()
    opt.zero_grad()
    m(x).square().sum().backward()
    opt.step()
    torch.cuda.synchronize()
    assert not torch.equal(before, m.W.vals), "the live weights did not move after pruning"
    # the Parameter keeps its handle alive even after the module lets go of it
    ref = weakref.ref(m.W)
    p = m.vals
    del m
    gc.collect()
    assert ref() is not None, "handle freed while its vals Parameter is alive"
    assert torch.isfinite(p.detach().sum())
    del p, p_before, opt
    gc.collect()
    assert ref() is None, "handle leaked after the last view died"


def test_first_call_under_no_grad_runs_the_probe():
    """the auto dispatcher's first call may come under no_grad."""
    from paper_2302_04852_b200.nn import SparseLinear
    c = synth.linear_case(256, 256, 64, 0.1, 1.0 / 256, 36)
    m = SparseLinear(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda(), mode="auto")
    x = torch.from_numpy(c["X"].T.copy()).cuda()
    with torch.no_grad():
        y = m(x)
    assert m.impl in ("sparse", "dense") and set(m.probe_ms) == {"dense", "sparse"}
    assert m.vals.grad is None
    with torch.inference_mode():
        y2 = m(x)
    torch.cuda.synchronize()
    assert torch.allclose(y, y2)


def test_conv_module_dispatch_times_both_sparse_kernels():
    """P427: at >= 80 % sparsity the NCHW conv module times dense, the batch-last
    sparse kernel and SparseConvOverON, keeps the fastest, and each of the three
    matches the float64 reference."""
    from paper_2302_04852_b200.nn import SparseConv2d
    c = synth.conv_case(OC=64, IC=64, H=28, W=28, KH=1, KW=1, pad=0, B=4, density=0.1, wvar=1.0 / 64, seed=41)
    Wt, Mt = torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda()
    x = torch.from_numpy(c["X"]).permute(3, 0, 1, 2).contiguous().cuda()
    ref = torch.nn.functional.conv2d(x.cpu().double(), (Wt * Mt).cpu().double(), padding=0)
    m = SparseConv2d(Wt, Mt, padding=0, mode="auto")
    y = m(x)
    assert set(m.probe_ms) == {"dense", "sparse", "sparse_nchw"}
    assert m.impl == min(m.probe_ms, key=m.probe_ms.get) or m.probe_ms[m.impl] <= min(m.probe_ms.values())
    _ok("auto", y, ref)
    for impl in ("dense", "sparse", "sparse_nchw"):
        mm = SparseConv2d(Wt, Mt, padding=0, mode=impl)
        _ok(impl, mm(x), ref)

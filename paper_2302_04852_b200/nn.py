"""Drop-in PyTorch modules over libsparseprop (the paper's "two Pytorch modules,
one for linear and one for convolution layers", P358 §4) and the §4.2
dense/sparse dispatcher (P427-P429).

`SparseLinear` / `SparseConv2d` hold their kept weights as a Parameter that IS
the handle's vals buffer (zero-copy), so any torch optimizer updates the
weights the kernels read.  Autograd runs the library's kernels: forward SpMM,
and the fused CSC-driven backward (dX and dW in one pass) -- dW is produced
only at the nonzeros.  Layouts: `SparseLinear` takes PyTorch's [N, in] inputs
(transposed to the kernels' batch-contiguous [in, N] internally) or, with
feature_major=True, [in, N] directly; `SparseConv2d` takes NCHW (permuted to
the kernels' CHWN) or, with batch_last=True, CHWN directly.

Dispatcher (P427-P429): a module less than 80 % sparse runs dense; at >= 80 %
the first forward+backward on a probe batch is timed both ways (CUDA events)
and the faster implementation is kept until the mask changes
(`set_mask`).  The dense path is a cuBLAS / cuDNN call on the densified
weight (sp_weight_to_dense) with its gradient restricted to the mask by
sp_weight_gather -- both libsparseprop kernels.  `timer` can be replaced
(tests use a fake one).
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from . import sparseprop as sp

DENSE_BELOW = 0.80  # P427: "dense ... as long as they are less than 80% sparse"


# ---------------------------------------------------------------------------
# autograd functions (feature-major / batch-last layouts; kernels only)
# ---------------------------------------------------------------------------
class _SparseLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, xt, vals, W):  # xt [in, N] contiguous
        ctx.W = W
        ctx.save_for_backward(xt)
        return sp.sp_linear_fwd(W, xt)

    @staticmethod
    def backward(ctx, gy):
        (xt,) = ctx.saved_tensors
        dX, dW = sp.sp_linear_bwd(ctx.W, xt, gy.contiguous())
        return dX, dW, None


class _DenseMaskedFn(torch.autograd.Function):
    """Dense path: y = W_dense @ x with W_dense = to_dense(vals); dvals = gather(dW_dense)."""

    @staticmethod
    def forward(ctx, xt, vals, W):
        Wd = W.to_dense(vals)
        ctx.W = W
        ctx.save_for_backward(xt, Wd)
        return Wd @ xt

    @staticmethod
    def backward(ctx, gy):
        xt, Wd = ctx.saved_tensors
        dX = Wd.t() @ gy
        dvals = sp.sp_weight_gather(ctx.W, gy @ xt.t())
        return dX, dvals, None


class _SparseConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, vals, W, g):  # x CHWN contiguous
        ctx.W, ctx.g = W, g
        ctx.save_for_backward(x)
        return sp.sp_conv2d_fwd(W, g, x)

    @staticmethod
    def backward(ctx, gy):
        (x,) = ctx.saved_tensors
        gy = gy.contiguous()
        dX, dW = sp.sp_conv2d_bwd(ctx.W, ctx.g, x, gy)  # both products in one pass (Alg. 2)
        return dX, dW, None, None


class _SparseConvNCHWFn(torch.autograd.Function):
    """The paper's SparseConvOverON (P293, P397): NCHW in and out, no permutes."""

    @staticmethod
    def forward(ctx, x, vals, W, g):  # x NCHW contiguous
        ctx.W, ctx.g = W, g
        ctx.save_for_backward(x)
        return sp.sp_conv2d_fwd_nchw(W, g, x)

    @staticmethod
    def backward(ctx, gy):
        (x,) = ctx.saved_tensors
        dX, dW = sp.sp_conv2d_bwd_nchw(ctx.W, ctx.g, x, gy.contiguous())
        return dX, dW, None, None


def _fp32_cudnn():
    """The dense path stays fp32 (P134): no TF32 tensor-core convolutions."""
    return torch.backends.cudnn.flags(enabled=True, benchmark=False, deterministic=False, allow_tf32=False)


class _DenseConvFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, vals, W, g):  # x CHWN
        Wd = W.to_dense(vals).view(W.filter_shape)
        xn = x.permute(3, 0, 1, 2)
        ctx.W, ctx.g = W, g
        ctx.save_for_backward(xn, Wd)
        with _fp32_cudnn():
            return F.conv2d(xn, Wd, padding=g.pad).permute(1, 2, 3, 0).contiguous()

    @staticmethod
    def backward(ctx, gy):
        xn, Wd = ctx.saved_tensors
        gyn = gy.permute(3, 0, 1, 2)
        with _fp32_cudnn():
            dxn = torch.nn.grad.conv2d_input(xn.shape, Wd, gyn, padding=ctx.g.pad)
            dWd = torch.nn.grad.conv2d_weight(xn, Wd.shape, gyn, padding=ctx.g.pad)
        dvals = sp.sp_weight_gather(ctx.W, dWd.reshape(Wd.shape[0], -1))
        return dxn.permute(1, 2, 3, 0).contiguous(), dvals, None, None


# ---------------------------------------------------------------------------
# dispatcher (P427-P429)
# ---------------------------------------------------------------------------
def cuda_timer(fn, reps: int = 3) -> float:
    """Device time (ms) of fn() on the current stream: CUDA events, the fastest
    of `reps` calls after two warm-ups (the first call of a kernel in a process
    pays its module load and the library's one-time pool setup)."""
    fn()
    fn()
    best = float("inf")
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def decide(sparsity: float, time_dense, time_sparse, mode: str = "auto", more_sparse: dict | None = None) -> str:
    """The §4.2 rule: forced modes win; below 80 % sparsity -> dense without
    probing; otherwise the fastest of one timed forward+backward of each
    implementation -- dense, sparse, and (convolution: "both sparse
    implementations are considered", P427) the extra sparse ones in
    `more_sparse` {name: timer}.  Ties go to the sparse implementations, in
    order."""
    names = ["sparse"] + list(more_sparse or {})
    if mode == "dense" or mode in names:
        return mode
    if sparsity < DENSE_BELOW:
        return "dense"
    timers = {"sparse": time_sparse, **(more_sparse or {})}
    best, best_t = "dense", time_dense()
    for n in reversed(names):  # ties: the first sparse implementation wins
        t = timers[n]()
        if t <= best_t:
            best, best_t = n, t
    return best


class _Dispatching(torch.nn.Module):
    def __init__(self, mode: str, timer):
        super().__init__()
        self.mode = mode
        self.timer = timer
        self.impl = None  # decided lazily on the first batch, reset by set_mask
        self.probe_ms = None

    def _rebuild(self, weight: torch.Tensor, mask: torch.Tensor):
        """New handle for (weight, mask).  The `vals` Parameter OBJECT is kept
        across mask changes (its .data is re-pointed at the new handle's vals,
        whose storage keeps that handle alive), so an optimizer built before a
        GMP update keeps stepping the live weights.  Its size changes with
        nnz: per-parameter optimizer state (momentum, Adam moments) must be
        dropped by the caller -- `prune.prune_modules(..., optimizer=opt)`
        does it."""
        self.W = sp.sp_weight_create(weight.detach().float().contiguous(), mask.to(torch.uint8).contiguous())
        if getattr(self, "vals", None) is None:
            self.vals = torch.nn.Parameter(self.W.vals, requires_grad=True)
        else:
            self.vals.data = self.W.vals
            self.vals.grad = None
        self.impl = None

    def _extra_impls(self):
        """Sparse implementations besides "sparse" the dispatcher times."""
        return []

    @property
    def sparsity(self) -> float:
        return 1.0 - self.W.nnz / float(self.W.R * self.W.C)

    def _choose(self, x):
        if self.impl is None:
            def run(fn):
                def go():
                    # the probe is a forward+backward even when the first call
                    # comes under no_grad / inference_mode (e.g. eval first)
                    with torch.inference_mode(False), torch.enable_grad():
                        xx = x.detach().clone().requires_grad_(x.requires_grad)
                        out = fn(xx)
                        out.backward(torch.ones_like(out))
                return lambda: self.timer(go)
            self.probe_ms = {}

            def td():
                self.probe_ms["dense"] = run(lambda xx: self._run(xx, "dense"))()
                return self.probe_ms["dense"]

            def ts():
                self.probe_ms["sparse"] = run(lambda xx: self._run(xx, "sparse"))()
                return self.probe_ms["sparse"]

            def timer_of(name):
                def t():
                    self.probe_ms[name] = run(lambda xx: self._run(xx, name))()
                    return self.probe_ms[name]
                return t
            extra = {n: timer_of(n) for n in self._extra_impls()}
            self.impl = decide(self.sparsity, td, ts, self.mode, extra)
            if self.vals.grad is not None:  # probes must not leak gradients
                self.vals.grad = None
        return self.impl


class SparseLinear(_Dispatching):
    """y = x W^T with W (out x in) restricted to a fixed mask (no bias)."""

    def __init__(self, weight: torch.Tensor, mask: torch.Tensor, feature_major: bool = False,
                 mode: str = "auto", timer=cuda_timer):
        super().__init__(mode, timer)
        self.feature_major = feature_major
        self.set_mask(weight, mask)

    def set_mask(self, weight: torch.Tensor, mask: torch.Tensor):
        """(Re)build the sparse structure (masks change "only a few times", P428)."""
        self._rebuild(weight, mask)

    def _run(self, x, impl):
        xt = x if self.feature_major else x.t()
        xt = xt.contiguous()
        fn = _SparseLinearFn if impl == "sparse" else _DenseMaskedFn
        y = fn.apply(xt, self.vals, self.W)
        return y if self.feature_major else y.t()

    def forward(self, x):
        return self._run(x, self._choose(x))


class SparseConv2d(_Dispatching):
    """Stride-1 conv with a fixed sparse filter [OC][IC][KH][KW] (no bias)."""

    def __init__(self, weight: torch.Tensor, mask: torch.Tensor, padding: int = 0, batch_last: bool = False,
                 mode: str = "auto", timer=cuda_timer):
        super().__init__(mode, timer)
        self.padding = padding
        self.batch_last = batch_last
        self.set_mask(weight, mask)

    def set_mask(self, weight: torch.Tensor, mask: torch.Tensor):
        self._rebuild(weight, mask)

    def _extra_impls(self):
        # NCHW input: the batch-last kernel (on permuted copies) and
        # SparseConvOverON (natural layout) are both candidates (P427)
        return [] if self.batch_last else ["sparse_nchw"]

    def _run(self, x, impl):
        if impl == "sparse_nchw":  # SparseConvOverON: NCHW in and out
            xn = x.contiguous()
            B, C, H, Wd = xn.shape
            g = sp.conv_geom(self.W, B, H, Wd, self.padding)
            return _SparseConvNCHWFn.apply(xn, self.vals, self.W, g)
        xc = x if self.batch_last else x.permute(1, 2, 3, 0)
        xc = xc.contiguous()
        C, H, Wd, B = xc.shape
        g = sp.conv_geom(self.W, B, H, Wd, self.padding)
        fn = _SparseConvFn if impl == "sparse" else _DenseConvFn
        y = fn.apply(xc, self.vals, self.W, g)
        return y if self.batch_last else y.permute(3, 0, 1, 2)

    def forward(self, x):
        return self._run(x, self._choose(x))

"""SparseProp oracle -- TEST INFRASTRUCTURE ONLY.

Plain fp64 CPU implementation of the hot path (§3.2-§3.3), used by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs ONLY.  The product (paper_2302_04852_b200) never imports this package and
the two share no code; both take their inputs from `synth`.

The arithmetic lives in sparseprop_oracle.c (plain loops, fp64); this module is
marshalling plus the cfg5 MLP composition (forward / MSE / backward), which is
written out here from the layer functions, numpy ReLU and the SURVEY C18 loss.
Every function cites the passage it follows; see the C file for the pins.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sparseprop_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

__all__ = [
    "build", "Csr", "csr_from_mask", "linear_fwd", "linear_bwd_input", "linear_bwd_weight",
    "densify", "ConvFormat", "conv_format", "conv2d_fwd", "conv2d_bwd", "chwn_to_nchw",
    "nchw_to_chwn", "mlp_step", "threads_available",
]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no -ffast-math, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ct.CDLL(build())
        i64, i32p, f64p, u8p = ct.c_int64, ct.POINTER(ct.c_int32), ct.POINTER(ct.c_double), \
            ct.POINTER(ct.c_uint8)
        _lib.or_mask_nnz.restype = i64
        _lib.or_conv_format.restype = i64
        _lib.or_csc_build.restype = ct.c_int
        _lib.or_num_threads_available.restype = ct.c_int
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(ct.POINTER(t))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def threads_available() -> int:
    return int(_L().or_num_threads_available())


class Csr:
    """The oracle's own CSR + CSC index copy (P153-P154, P183)."""

    def __init__(self, R, C, row_ptr, col_idx, vals, col_ptr, row_idx, perm):
        self.R, self.C = R, C
        self.row_ptr, self.col_idx, self.vals = row_ptr, col_idx, vals
        self.col_ptr, self.row_idx, self.perm = col_ptr, row_idx, perm

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def with_vals(self, vals) -> "Csr":
        return Csr(self.R, self.C, self.row_ptr, self.col_idx, _f64(vals), self.col_ptr,
                   self.row_idx, self.perm)


def csr_from_mask(dense, mask) -> Csr:
    """CSR (structure = mask, C10) + CSC index copy with perm (C11, C23)."""
    L = _L()
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    R, C = mask.shape
    dense = _f64(dense).reshape(R, C)
    nnz = int(L.or_mask_nnz(ct.c_int64(R), ct.c_int64(C), _p(mask, ct.c_uint8)))
    row_ptr = np.zeros(R + 1, np.int32)
    col_idx = np.zeros(max(nnz, 1), np.int32)
    vals = np.zeros(max(nnz, 1), np.float64)
    L.or_csr_build(ct.c_int64(R), ct.c_int64(C), _p(mask, ct.c_uint8), _p(dense, ct.c_double),
                   _p(row_ptr, ct.c_int32), _p(col_idx, ct.c_int32), _p(vals, ct.c_double))
    col_ptr = np.zeros(C + 1, np.int32)
    row_idx = np.zeros(max(nnz, 1), np.int32)
    perm = np.zeros(max(nnz, 1), np.int32)
    rc = L.or_csc_build(ct.c_int64(R), ct.c_int64(C), _p(mask, ct.c_uint8),
                        _p(col_ptr, ct.c_int32), _p(row_idx, ct.c_int32), _p(perm, ct.c_int32))
    if rc != 0:
        raise MemoryError("oracle csc build")
    return Csr(R, C, row_ptr, col_idx[:nnz], vals[:nnz], col_ptr, row_idx[:nnz], perm[:nnz])


def linear_fwd(W: Csr, X, nthreads: int = 1) -> np.ndarray:
    """Y = W X (P141, orientation per SURVEY C1); X [C x B] -> Y [R x B], fp64."""
    X = _f64(X)
    B = X.shape[1]
    assert X.shape[0] == W.C
    Y = np.empty((W.R, B), np.float64)
    _L().or_linear_fwd(ct.c_int64(W.R), ct.c_int64(B), _p(W.row_ptr, ct.c_int32),
                       _p(W.col_idx, ct.c_int32), _p(_f64(W.vals), ct.c_double),
                       _p(X, ct.c_double), _p(Y, ct.c_double), ct.c_int(nthreads))
    return Y


def linear_bwd_input(W: Csr, dY, nthreads: int = 1) -> np.ndarray:
    """dX = W^T dY (Eq. 1, P143-P145) via the CSC copy; [R x B] -> [C x B]."""
    dY = _f64(dY)
    B = dY.shape[1]
    assert dY.shape[0] == W.R
    dX = np.empty((W.C, B), np.float64)
    _L().or_linear_bwd_input(ct.c_int64(W.C), ct.c_int64(B), _p(W.col_ptr, ct.c_int32),
                             _p(W.row_idx, ct.c_int32), _p(W.perm, ct.c_int32),
                             _p(_f64(W.vals), ct.c_double), _p(dY, ct.c_double),
                             _p(dX, ct.c_double), ct.c_int(nthreads))
    return dX


def linear_bwd_weight(W: Csr, X, dY, nthreads: int = 1) -> np.ndarray:
    """dW = (dY X^T) restricted to the mask (Eq. 2, P146-P148, SDDMM P151),
    nnz-length in CSR order."""
    X, dY = _f64(X), _f64(dY)
    B = X.shape[1]
    assert X.shape == (W.C, B) and dY.shape == (W.R, B)
    dW = np.empty(W.nnz, np.float64)
    _L().or_linear_bwd_weight(ct.c_int64(W.R), ct.c_int64(B), _p(W.row_ptr, ct.c_int32),
                              _p(W.col_idx, ct.c_int32), _p(X, ct.c_double),
                              _p(dY, ct.c_double), _p(dW, ct.c_double), ct.c_int(nthreads))
    return dW


def densify(W: Csr, nz) -> np.ndarray:
    """Scatter an nnz buffer over the CSR support; exact +0.0 elsewhere."""
    out = np.empty((W.R, W.C), np.float64)
    _L().or_densify(ct.c_int64(W.R), ct.c_int64(W.C), _p(W.row_ptr, ct.c_int32),
                    _p(W.col_idx, ct.c_int32), _p(_f64(nz), ct.c_double), _p(out, ct.c_double))
    return out


class ConvFormat:
    """The paper's 4-array sparse conv format (P251): och, ich, x, y, vals."""

    def __init__(self, OC, IC, KH, KW, och, ich, wx, wy, vals):
        self.OC, self.IC, self.KH, self.KW = OC, IC, KH, KW
        self.och, self.ich, self.wx, self.wy, self.vals = och, ich, wx, wy, vals

    @property
    def nnz(self) -> int:
        return int(self.och[-1])


def conv_format(dense, mask) -> ConvFormat:
    """Build the 4-array format from [OC][IC][KH][KW] dense + mask (P251-P285)."""
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    OC, IC, KH, KW = mask.shape
    dense = _f64(dense).reshape(mask.shape)
    nmax = max(int(mask.astype(bool).sum()), 1)
    och = np.zeros(OC + 1, np.int32)
    ich = np.zeros(OC * (IC + 1), np.int32)
    wx = np.zeros(nmax, np.int32)
    wy = np.zeros(nmax, np.int32)
    vals = np.zeros(nmax, np.float64)
    n = int(_L().or_conv_format(ct.c_int64(OC), ct.c_int64(IC), ct.c_int64(KH), ct.c_int64(KW),
                                _p(mask, ct.c_uint8), _p(dense, ct.c_double),
                                _p(och, ct.c_int32), _p(ich, ct.c_int32), _p(wx, ct.c_int32),
                                _p(wy, ct.c_int32), _p(vals, ct.c_double)))
    return ConvFormat(OC, IC, KH, KW, och, ich, wx[:n], wy[:n], vals[:n])


def conv2d_fwd(F: ConvFormat, X_nchw, pad: int, nthreads: int = 1) -> np.ndarray:
    """Eq. (3) with padding (P224-P229), NCHW fp64."""
    X = _f64(X_nchw)
    B, IC, M, N = X.shape
    assert IC == F.IC
    OM, ON = M + 2 * pad - F.KH + 1, N + 2 * pad - F.KW + 1
    O = np.empty((B, F.OC, OM, ON), np.float64)
    _L().or_conv2d_fwd(ct.c_int64(B), ct.c_int64(IC), ct.c_int64(M), ct.c_int64(N),
                       ct.c_int64(F.OC), ct.c_int64(F.KH), ct.c_int64(F.KW), ct.c_int64(pad),
                       _p(F.och, ct.c_int32), _p(F.ich, ct.c_int32), _p(F.wx, ct.c_int32),
                       _p(F.wy, ct.c_int32), _p(_f64(F.vals), ct.c_double), _p(X, ct.c_double),
                       _p(O, ct.c_double), ct.c_int(nthreads))
    return O


def conv2d_bwd(F: ConvFormat, X_nchw, dO_nchw, pad: int):
    """Algorithm 2 (P297-P347, readings C5/C6): returns (dX NCHW, dW nnz in
    (oc, ic, x, y) order == CSR order of the flattened filter)."""
    X, dO = _f64(X_nchw), _f64(dO_nchw)
    B, IC, M, N = X.shape
    OM, ON = M + 2 * pad - F.KH + 1, N + 2 * pad - F.KW + 1
    assert dO.shape == (B, F.OC, OM, ON)
    dX = np.empty_like(X)
    dW = np.empty(F.nnz, np.float64)
    _L().or_conv2d_bwd(ct.c_int64(B), ct.c_int64(IC), ct.c_int64(M), ct.c_int64(N),
                       ct.c_int64(F.OC), ct.c_int64(F.KH), ct.c_int64(F.KW), ct.c_int64(pad),
                       _p(F.och, ct.c_int32), _p(F.ich, ct.c_int32), _p(F.wx, ct.c_int32),
                       _p(F.wy, ct.c_int32), _p(_f64(F.vals), ct.c_double), _p(X, ct.c_double),
                       _p(dO, ct.c_double), _p(dX, ct.c_double), _p(dW, ct.c_double))
    return dX, dW


def chwn_to_nchw(a):
    """Exact layout permutation [C][H][W][B] -> [B][C][H][W]."""
    return np.ascontiguousarray(np.transpose(a, (3, 0, 1, 2)))


def nchw_to_chwn(a):
    return np.ascontiguousarray(np.transpose(a, (1, 2, 3, 0)))


def mlp_step(layers, X0, target, nthreads: int = 1):
    """One cfg5 step on the full batch (north star).

    layers: list of (Csr W1, Csr W2) per block, W1 d_ff x d_model, W2 d_model x d_ff.
    Forward per block: Z = W1 X, H = max(Z, 0), X' = W2 H.
    Loss L = 1/2 sum (Y - T)^2 (C18); dY = Y - T.
    Backward per block (reverse): dW2 = SDDMM(H, dY), dH = W2^T dY,
    dZ = dH * [H > 0] (C26: ReLU'(0) = 0), dW1 = SDDMM(X, dZ), dX = W1^T dZ.
    Returns dict(loss, Y, dW=[(dW1, dW2)...], acts=[(X_l, H_l)...], dX0,
    dYs=[(dZ_l, dY_l)...]) -- the saved tensors feed the layer-local parity
    protocol (C19).
    """
    X = _f64(X0)
    acts = []
    for (W1, W2) in layers:
        Z = linear_fwd(W1, X, nthreads)
        H = np.maximum(Z, 0.0)
        acts.append((X, H))
        X = linear_fwd(W2, H, nthreads)
    Y = X
    diff = Y - _f64(target)
    loss = 0.5 * float(np.sum(diff * diff))
    dY = diff
    dWs = [None] * len(layers)
    dYs = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        W1, W2 = layers[l]
        Xl, Hl = acts[l]
        dW2 = linear_bwd_weight(W2, Hl, dY, nthreads)
        dH = linear_bwd_input(W2, dY, nthreads)
        dZ = dH * (Hl > 0.0)
        dW1 = linear_bwd_weight(W1, Xl, dZ, nthreads)
        dYs[l] = (dZ, dY)
        dY = linear_bwd_input(W1, dZ, nthreads)
        dWs[l] = (dW1, dW2)
    return dict(loss=loss, Y=Y, dW=dWs, acts=acts, dX0=dY, dYs=dYs)

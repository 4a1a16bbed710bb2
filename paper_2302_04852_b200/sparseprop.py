"""Thin ctypes binding of libsparseprop (include/sparseprop.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of csrc/.  Tensors are torch CUDA tensors (fp32 / uint8 / int32,
contiguous); streams default to torch's current stream.  There is NO CPU
fallback: without the built library or a CUDA device every call raises.

Function names are the C names; `SparseWeight` is a convenience owner of an
sp_weight_t handle.
"""
from __future__ import annotations

import ctypes as ct
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPARSEPROP_LIB") or os.path.join(_HERE, "libsparseprop.so")  # override: A/B builds

SP_STATUS = {0: "SP_OK", 1: "SP_ERR_NULL", 2: "SP_ERR_SHAPE", 3: "SP_ERR_OVERFLOW",
             4: "SP_ERR_ALLOC", 5: "SP_ERR_CUDA", 6: "SP_ERR_BAD_HANDLE"}

# every symbol include/sparseprop.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "sp_weight_create", "sp_weight_destroy", "sp_weight_nnz", "sp_weight_rows", "sp_weight_cols",
    "sp_weight_vals", "sp_weight_indices", "sp_weight_to_dense", "sp_linear_fwd",
    "sp_linear_bwd_input", "sp_linear_bwd_weight", "sp_linear_fwd_relu",
    "sp_linear_bwd_input_relu", "sp_conv2d_fwd", "sp_conv2d_bwd_input", "sp_conv2d_bwd_weight",
    "sp_mse_scratch_floats", "sp_mse_grad", "sp_sgd", "sp_last_error", "sp_version",
    "sp_launch_count", "sp_linear_bwd", "sp_linear_bwd_relu", "sp_weight_create_conv", "sp_weight_gather",
    "sp_weight_set_managed", "sp_weight_sgd",
    "sp_conv2d_bwd", "sp_set_sm_reserve", "sp_last_path",
    "sp_conv2d_fwd_nchw", "sp_conv2d_bwd_input_nchw", "sp_conv2d_bwd_weight_nchw", "sp_conv2d_bwd_nchw",
    "sp_comm_create", "sp_comm_open", "sp_comm_buffer", "sp_comm_allreduce", "sp_comm_ctas", "sp_comm_destroy",
    "sp_comm_create_local", "sp_comm_local_buffer", "sp_comm_allreduce_as", "sp_weights_sgd",
    "sp_nvls_supported", "sp_nvls_create", "sp_nvls_open", "sp_nvls_bind", "sp_nvls_buffer", "sp_nvls_allreduce",
    "sp_nvls_ctas", "sp_nvls_destroy",
]


class SparsePropError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{SP_STATUS.get(status, status)}: {msg}")
        self.status = status


class sp_conv_geom(ct.Structure):
    _fields_ = [(n, ct.c_int32) for n in ("B", "C_in", "H", "W", "C_out", "KH", "KW", "pad")]


_lib = None


def lib() -> ct.CDLL:
    """Load libsparseprop.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (no CPU fallback exists)")
        L = ct.CDLL(LIB_PATH)
        vp, i64, st = ct.c_void_p, ct.c_int64, ct.c_int
        sig = {
            "sp_weight_create": (st, [i64, i64, vp, vp, vp, ct.POINTER(vp)]),
            "sp_weight_destroy": (st, [vp, vp]),
            "sp_weight_nnz": (i64, [vp]), "sp_weight_rows": (i64, [vp]), "sp_weight_cols": (i64, [vp]),
            "sp_weight_vals": (st, [vp, ct.POINTER(vp)]),
            "sp_weight_indices": (st, [vp] + [ct.POINTER(vp)] * 5),
            "sp_weight_to_dense": (st, [vp, vp, vp, vp]),
            "sp_weight_gather": (st, [vp, vp, vp, vp]),
            "sp_linear_fwd": (st, [vp, vp, vp, i64, vp]),
            "sp_linear_fwd_relu": (st, [vp, vp, vp, i64, vp]),
            "sp_linear_bwd_input": (st, [vp, vp, vp, i64, vp]),
            "sp_linear_bwd_input_relu": (st, [vp, vp, vp, vp, i64, vp]),
            "sp_linear_bwd_weight": (st, [vp, vp, vp, vp, i64, vp]),
            "sp_conv2d_fwd": (st, [vp, ct.POINTER(sp_conv_geom), vp, vp, vp]),
            "sp_conv2d_bwd_input": (st, [vp, ct.POINTER(sp_conv_geom), vp, vp, vp]),
            "sp_conv2d_bwd_weight": (st, [vp, ct.POINTER(sp_conv_geom), vp, vp, vp, vp]),
            "sp_conv2d_bwd": (st, [vp, ct.POINTER(sp_conv_geom), vp, vp, vp, vp, vp]),
            "sp_mse_scratch_floats": (i64, [i64]),
            "sp_mse_grad": (st, [vp, vp, vp, vp, vp, i64, vp]),
            "sp_sgd": (st, [vp, vp, i64, ct.c_float, vp]),
            "sp_last_error": (ct.c_char_p, []),
            "sp_version": (ct.c_char_p, []),
            "sp_launch_count": (ct.c_uint64, []),
            "sp_linear_bwd": (st, [vp, vp, vp, vp, vp, i64, vp]),
            "sp_weight_create_conv": (st, [ct.c_int32] * 4 + [vp, vp, vp, ct.POINTER(vp)]),
            "sp_linear_bwd_relu": (st, [vp, vp, vp, vp, vp, vp, i64, vp]),
            "sp_weight_set_managed": (st, [vp, ct.c_int]),
            "sp_weight_sgd": (st, [vp, vp, ct.c_float, vp]),
            "sp_set_sm_reserve": (st, [ct.c_int32]),
            "sp_last_path": (ct.c_char_p, []),
            "sp_conv2d_fwd_nchw": (st, [vp, ct.POINTER(sp_conv_geom), vp, vp, vp]),
            "sp_conv2d_bwd_input_nchw": (st, [vp, ct.POINTER(sp_conv_geom), vp, vp, vp]),
            "sp_conv2d_bwd_weight_nchw": (st, [vp, ct.POINTER(sp_conv_geom), vp, vp, vp, vp]),
            "sp_conv2d_bwd_nchw": (st, [vp, ct.POINTER(sp_conv_geom), vp, vp, vp, vp, vp]),
            "sp_weights_sgd": (st, [ct.POINTER(vp), ct.POINTER(vp), ct.c_int32, ct.c_float, vp]),
            "sp_comm_create": (st, [ct.c_int32, ct.c_int32, i64, ct.POINTER(vp), vp]),
            "sp_comm_open": (st, [vp, vp]),
            "sp_comm_buffer": (vp, [vp]),
            "sp_comm_allreduce": (st, [vp, i64, i64, vp]),
            "sp_comm_ctas": (ct.c_int32, []),
            "sp_comm_destroy": (st, [vp]),
            "sp_comm_create_local": (st, [ct.c_int32, i64, ct.POINTER(vp)]),
            "sp_comm_local_buffer": (vp, [vp, ct.c_int32]),
            "sp_comm_allreduce_as": (st, [vp, ct.c_int32, i64, i64, vp]),
            "sp_nvls_supported": (ct.c_int32, []),
            "sp_nvls_create": (st, [ct.c_int32, ct.c_int32, i64, ct.POINTER(vp), ct.POINTER(ct.c_int32)]),
            "sp_nvls_open": (st, [vp, ct.c_int32]),
            "sp_nvls_bind": (st, [vp]),
            "sp_nvls_buffer": (vp, [vp]),
            "sp_nvls_allreduce": (st, [vp, i64, i64, vp]),
            "sp_nvls_ctas": (ct.c_int32, []),
            "sp_nvls_destroy": (st, [vp]),
        }
        for name, (res, args) in sig.items():
            if os.environ.get("SPARSEPROP_LIB") and not hasattr(L, name):
                continue  # an A/B library built from older sources (tools/build_at_commit.py)
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise SparsePropError(status, lib().sp_last_error().decode())


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if isinstance(stream, torch.cuda.Stream) else int(stream)


def _dev(t: torch.Tensor, dtype, name: str) -> int:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor (libsparseprop has no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    return t.data_ptr()


def version() -> str:
    return lib().sp_version().decode()


def last_path() -> str:
    """Kernel families the last compute call on this thread launched (provenance)."""
    return lib().sp_last_path().decode()


def launch_count() -> int:
    """Kernels launched by libsparseprop so far in this process."""
    return int(lib().sp_launch_count())


class SparseWeight:
    """Owner of an sp_weight_t: CSR + CSC index copy + vals, all on the device."""

    def __init__(self, dense: torch.Tensor, mask: torch.Tensor, stream=None):
        if dense.dim() == 4:  # conv filter [OC][IC][KH][KW]
            self.filter_shape = tuple(dense.shape)
            dense = dense.reshape(dense.shape[0], -1)
            mask = mask.reshape(mask.shape[0], -1)
        else:
            self.filter_shape = None
        if dense.dim() != 2 or dense.shape != mask.shape:
            raise ValueError("dense and mask must be R x C (or matching 4-D conv filters)")
        R, C = dense.shape
        h = ct.c_void_p()
        # the contiguous copies stay bound to locals until the C call returns: a
        # temporary freed inside _dev could be handed to the next copy by the
        # caching allocator and overwritten before the library reads it
        d = dense.contiguous()
        m = mask.contiguous()
        if self.filter_shape is not None:
            OC, IC, KH, KW = self.filter_shape
            _check(lib().sp_weight_create_conv(OC, IC, KH, KW, _dev(d, torch.float32, "dense"),
                                               _dev(m, torch.uint8, "mask"), _stream(stream), ct.byref(h)))
        else:
            _check(lib().sp_weight_create(R, C, _dev(d, torch.float32, "dense"), _dev(m, torch.uint8, "mask"),
                                          _stream(stream), ct.byref(h)))
        del d, m
        self.handle = h
        self.R, self.C = int(R), int(C)
        self.nnz = int(lib().sp_weight_nnz(h))
        self.device = dense.device
        p = ct.c_void_p()
        _check(lib().sp_weight_vals(h, ct.byref(p)))
        self._vals_ptr = p.value

    # -- zero-copy views of the handle-owned device buffers ------------------
    def _view(self, ptr: int, n: int, dtype) -> torch.Tensor:
        """A tensor over handle-owned device memory.  torch keeps the
        __cuda_array_interface__ object alive for the storage's lifetime, and
        that object holds this SparseWeight: every tensor sharing the storage
        (views, nn.Parameter aliases, optimizer references) keeps the handle
        alive, and the handle is destroyed only after the last of them dies.
        No reference runs back from the handle to its views (no cycle)."""
        if n == 0:
            return torch.empty(0, dtype=dtype, device=self.device)
        typestr = {torch.float32: "<f4", torch.int32: "<i4"}[dtype]

        class _CAI:
            def __init__(self, owner):
                self.owner = owner
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                                 "version": 3, "strides": None, "stream": None}
        return torch.as_tensor(_CAI(self), device=self.device)

    @property
    def vals(self) -> torch.Tensor:
        """Mutable fp32 view of vals[nnz] (CSR order), zero-copy; keeps the handle alive."""
        return self._view(self._vals_ptr, self.nnz, torch.float32)

    def indices(self) -> dict:
        ps = [ct.c_void_p() for _ in range(5)]
        _check(lib().sp_weight_indices(self.handle, *[ct.byref(p) for p in ps]))
        names = ["row_ptr", "col_idx", "col_ptr", "row_idx", "perm"]
        sizes = [self.R + 1, self.nnz, self.C + 1, self.nnz, self.nnz]
        return {n: self._view(p.value, s, torch.int32) for n, p, s in zip(names, ps, sizes)}

    def to_dense(self, nz: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        nz = self.vals if nz is None else nz
        out = torch.empty(self.R, self.C, dtype=torch.float32, device=self.device)
        sp_weight_to_dense(self, nz, out, stream)
        return out

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().sp_weight_destroy(self.handle, _stream(None))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# C-named wrappers (argument marshalling only)
# ---------------------------------------------------------------------------
def sp_weight_create(dense: torch.Tensor, mask: torch.Tensor, stream=None) -> SparseWeight:
    return SparseWeight(dense, mask, stream)


def sp_weight_to_dense(W: SparseWeight, nz: torch.Tensor, out: torch.Tensor, stream=None):
    _check(lib().sp_weight_to_dense(W.handle, _dev(nz, torch.float32, "nz") if W.nnz else None,
                                    _dev(out, torch.float32, "out"), _stream(stream)))
    return out


def sp_weight_gather(W: SparseWeight, dense: torch.Tensor, nz: torch.Tensor | None = None, stream=None):
    """nz[j] = dense[r_j][c_j] (restrict a dense R x C tensor to the mask)."""
    if nz is None:
        nz = torch.empty(W.nnz, dtype=torch.float32, device=dense.device)
    if tuple(dense.shape[-2:]) != (W.R, W.C) and dense.numel() != W.R * W.C:
        raise ValueError("dense must hold R x C values")
    d = dense.contiguous()  # bound until the (stream-ordered) call is enqueued
    if nz.numel() != W.nnz:
        raise ValueError("nz must have nnz elements")
    _check(lib().sp_weight_gather(W.handle, _dev(d, torch.float32, "dense"),
                                  _dev(nz, torch.float32, "nz") if W.nnz else None, _stream(stream)))
    if stream is not None and d is not dense:  # the copy must outlive the enqueued kernel
        d.record_stream(stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.ExternalStream(int(stream)))
    return nz


def _B(t: torch.Tensor, rows: int, name: str) -> int:
    if t.dim() != 2 or t.shape[0] != rows:
        raise ValueError(f"{name}: expected [{rows} x B], got {tuple(t.shape)}")
    return int(t.shape[1])


def sp_linear_fwd(W: SparseWeight, X: torch.Tensor, Y: torch.Tensor | None = None, stream=None,
                  relu: bool = False) -> torch.Tensor:
    B = _B(X, W.C, "X")
    if Y is None:
        Y = torch.empty(W.R, B, dtype=torch.float32, device=X.device)
    _B(Y, W.R, "Y")
    f = lib().sp_linear_fwd_relu if relu else lib().sp_linear_fwd
    _check(f(W.handle, _dev(X, torch.float32, "X"), _dev(Y, torch.float32, "Y"), B, _stream(stream)))
    return Y


def sp_linear_fwd_relu(W, X, Y=None, stream=None):
    return sp_linear_fwd(W, X, Y, stream, relu=True)


def sp_linear_bwd_input(W: SparseWeight, dY: torch.Tensor, dX: torch.Tensor | None = None,
                        stream=None, H: torch.Tensor | None = None) -> torch.Tensor:
    B = _B(dY, W.R, "dY")
    if dX is None:
        dX = torch.empty(W.C, B, dtype=torch.float32, device=dY.device)
    _B(dX, W.C, "dX")
    if H is None:
        _check(lib().sp_linear_bwd_input(W.handle, _dev(dY, torch.float32, "dY"),
                                         _dev(dX, torch.float32, "dX"), B, _stream(stream)))
    else:
        _B(H, W.C, "H")
        _check(lib().sp_linear_bwd_input_relu(W.handle, _dev(dY, torch.float32, "dY"),
                                              _dev(H, torch.float32, "H"),
                                              _dev(dX, torch.float32, "dX"), B, _stream(stream)))
    return dX


def sp_linear_bwd_input_relu(W, dY, H, dX=None, stream=None):
    return sp_linear_bwd_input(W, dY, dX, stream, H=H)


def sp_linear_bwd_weight(W: SparseWeight, X: torch.Tensor, dY: torch.Tensor,
                         dW: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    B = _B(X, W.C, "X")
    if _B(dY, W.R, "dY") != B:
        raise ValueError("X and dY batch sizes differ")
    if dW is None:
        dW = torch.empty(W.nnz, dtype=torch.float32, device=X.device)
    if dW.numel() != W.nnz:
        raise ValueError("dW must have nnz elements")
    _check(lib().sp_linear_bwd_weight(W.handle, _dev(X, torch.float32, "X"),
                                      _dev(dY, torch.float32, "dY"),
                                      _dev(dW, torch.float32, "dW") if W.nnz else None, B,
                                      _stream(stream)))
    return dW


def sp_linear_bwd(W: SparseWeight, X: torch.Tensor, dY: torch.Tensor, dX: torch.Tensor | None = None,
                  dW: torch.Tensor | None = None, stream=None, H: torch.Tensor | None = None):
    """Fused backward: (dX = W^T dY [* (H > 0)], dW = SDDMM(dY, X)) in one pass."""
    B = _B(X, W.C, "X")
    if _B(dY, W.R, "dY") != B:
        raise ValueError("X and dY batch sizes differ")
    if dX is None:
        dX = torch.empty(W.C, B, dtype=torch.float32, device=X.device)
    _B(dX, W.C, "dX")
    if dW is None:
        dW = torch.empty(W.nnz, dtype=torch.float32, device=X.device)
    if dW.numel() != W.nnz:
        raise ValueError("dW must have nnz elements")
    dwp = _dev(dW, torch.float32, "dW") if W.nnz else None
    if H is None:
        _check(lib().sp_linear_bwd(W.handle, _dev(X, torch.float32, "X"), _dev(dY, torch.float32, "dY"),
                                   _dev(dX, torch.float32, "dX"), dwp, B, _stream(stream)))
    else:
        _B(H, W.C, "H")
        _check(lib().sp_linear_bwd_relu(W.handle, _dev(X, torch.float32, "X"), _dev(dY, torch.float32, "dY"),
                                        _dev(H, torch.float32, "H"), _dev(dX, torch.float32, "dX"), dwp, B,
                                        _stream(stream)))
    return dX, dW


def sp_linear_bwd_relu(W, X, dY, H, dX=None, dW=None, stream=None):
    return sp_linear_bwd(W, X, dY, dX, dW, stream, H=H)


def conv_geom(W: SparseWeight, B: int, H: int, Wd: int, pad: int) -> sp_conv_geom:
    if W.filter_shape is None:
        raise ValueError("handle was not created from a 4-D conv filter")
    OC, IC, KH, KW = W.filter_shape
    return sp_conv_geom(B, IC, H, Wd, OC, KH, KW, pad)


def _geo_out(g: sp_conv_geom):
    return g.H + 2 * g.pad - g.KH + 1, g.W + 2 * g.pad - g.KW + 1


def _chk_shape(t: torch.Tensor, shape, name: str):
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")


def _chk_nnz(W: SparseWeight, dW: torch.Tensor, name: str = "dW"):
    if dW.numel() != W.nnz:
        raise ValueError(f"{name} must have nnz = {W.nnz} elements, got {dW.numel()}")


def sp_conv2d_fwd(W: SparseWeight, g: sp_conv_geom, X: torch.Tensor, Y: torch.Tensor | None = None,
                  stream=None) -> torch.Tensor:
    OH, OW = _geo_out(g)
    _chk_shape(X, (g.C_in, g.H, g.W, g.B), "X (CHWN [C_in][H][W][B])")
    if Y is None:
        Y = torch.empty(g.C_out, OH, OW, g.B, dtype=torch.float32, device=X.device)
    _chk_shape(Y, (g.C_out, OH, OW, g.B), "Y (CHWN [C_out][OH][OW][B])")
    _check(lib().sp_conv2d_fwd(W.handle, ct.byref(g), _dev(X, torch.float32, "X"),
                               _dev(Y, torch.float32, "Y"), _stream(stream)))
    return Y


def sp_conv2d_bwd_input(W: SparseWeight, g: sp_conv_geom, dY: torch.Tensor,
                        dX: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    OH, OW = _geo_out(g)
    _chk_shape(dY, (g.C_out, OH, OW, g.B), "dY (CHWN [C_out][OH][OW][B])")
    if dX is None:
        dX = torch.empty(g.C_in, g.H, g.W, g.B, dtype=torch.float32, device=dY.device)
    _chk_shape(dX, (g.C_in, g.H, g.W, g.B), "dX (CHWN [C_in][H][W][B])")
    _check(lib().sp_conv2d_bwd_input(W.handle, ct.byref(g), _dev(dY, torch.float32, "dY"),
                                     _dev(dX, torch.float32, "dX"), _stream(stream)))
    return dX


def sp_conv2d_bwd(W: SparseWeight, g: sp_conv_geom, X: torch.Tensor, dY: torch.Tensor,
                  dX: torch.Tensor | None = None, dW: torch.Tensor | None = None, stream=None):
    """Both conv backward products in one pass (Alg. 2 single pass): (dX, dW)."""
    OH, OW = _geo_out(g)
    _chk_shape(X, (g.C_in, g.H, g.W, g.B), "X (CHWN [C_in][H][W][B])")
    _chk_shape(dY, (g.C_out, OH, OW, g.B), "dY (CHWN [C_out][OH][OW][B])")
    if dX is None:
        dX = torch.empty(g.C_in, g.H, g.W, g.B, dtype=torch.float32, device=dY.device)
    _chk_shape(dX, (g.C_in, g.H, g.W, g.B), "dX (CHWN [C_in][H][W][B])")
    if dW is None:
        dW = torch.empty(W.nnz, dtype=torch.float32, device=X.device)
    _chk_nnz(W, dW)
    _check(lib().sp_conv2d_bwd(W.handle, ct.byref(g), _dev(X, torch.float32, "X"), _dev(dY, torch.float32, "dY"),
                               _dev(dX, torch.float32, "dX"), _dev(dW, torch.float32, "dW") if W.nnz else None,
                               _stream(stream)))
    return dX, dW


def sp_conv2d_bwd_weight(W: SparseWeight, g: sp_conv_geom, X: torch.Tensor, dY: torch.Tensor,
                         dW: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    OH, OW = _geo_out(g)
    _chk_shape(X, (g.C_in, g.H, g.W, g.B), "X (CHWN [C_in][H][W][B])")
    _chk_shape(dY, (g.C_out, OH, OW, g.B), "dY (CHWN [C_out][OH][OW][B])")
    if dW is None:
        dW = torch.empty(W.nnz, dtype=torch.float32, device=X.device)
    _chk_nnz(W, dW)
    _check(lib().sp_conv2d_bwd_weight(W.handle, ct.byref(g), _dev(X, torch.float32, "X"),
                                      _dev(dY, torch.float32, "dY"),
                                      _dev(dW, torch.float32, "dW") if W.nnz else None,
                                      _stream(stream)))
    return dW


# ---- NCHW (SparseConvOverON, P293 / P397): X, dX [B][C_in][H][W]; Y, dY [B][C_out][OH][OW]
def sp_conv2d_fwd_nchw(W: SparseWeight, g: sp_conv_geom, X: torch.Tensor, Y: torch.Tensor | None = None,
                       stream=None) -> torch.Tensor:
    OH, OW = _geo_out(g)
    _chk_shape(X, (g.B, g.C_in, g.H, g.W), "X (NCHW [B][C_in][H][W])")
    if Y is None:
        Y = torch.empty(g.B, g.C_out, OH, OW, dtype=torch.float32, device=X.device)
    _chk_shape(Y, (g.B, g.C_out, OH, OW), "Y (NCHW [B][C_out][OH][OW])")
    _check(lib().sp_conv2d_fwd_nchw(W.handle, ct.byref(g), _dev(X, torch.float32, "X"),
                                    _dev(Y, torch.float32, "Y"), _stream(stream)))
    return Y


def sp_conv2d_bwd_input_nchw(W: SparseWeight, g: sp_conv_geom, dY: torch.Tensor, dX: torch.Tensor | None = None,
                             stream=None) -> torch.Tensor:
    OH, OW = _geo_out(g)
    _chk_shape(dY, (g.B, g.C_out, OH, OW), "dY (NCHW [B][C_out][OH][OW])")
    if dX is None:
        dX = torch.empty(g.B, g.C_in, g.H, g.W, dtype=torch.float32, device=dY.device)
    _chk_shape(dX, (g.B, g.C_in, g.H, g.W), "dX (NCHW [B][C_in][H][W])")
    _check(lib().sp_conv2d_bwd_input_nchw(W.handle, ct.byref(g), _dev(dY, torch.float32, "dY"),
                                          _dev(dX, torch.float32, "dX"), _stream(stream)))
    return dX


def sp_conv2d_bwd_nchw(W: SparseWeight, g: sp_conv_geom, X: torch.Tensor, dY: torch.Tensor,
                       dX: torch.Tensor | None = None, dW: torch.Tensor | None = None, stream=None):
    """Both NCHW conv backward products in one pass: (dX, dW)."""
    OH, OW = _geo_out(g)
    _chk_shape(X, (g.B, g.C_in, g.H, g.W), "X (NCHW [B][C_in][H][W])")
    _chk_shape(dY, (g.B, g.C_out, OH, OW), "dY (NCHW [B][C_out][OH][OW])")
    if dX is None:
        dX = torch.empty(g.B, g.C_in, g.H, g.W, dtype=torch.float32, device=dY.device)
    _chk_shape(dX, (g.B, g.C_in, g.H, g.W), "dX (NCHW [B][C_in][H][W])")
    if dW is None:
        dW = torch.empty(W.nnz, dtype=torch.float32, device=X.device)
    _chk_nnz(W, dW)
    _check(lib().sp_conv2d_bwd_nchw(W.handle, ct.byref(g), _dev(X, torch.float32, "X"),
                                    _dev(dY, torch.float32, "dY"), _dev(dX, torch.float32, "dX"),
                                    _dev(dW, torch.float32, "dW") if W.nnz else None, _stream(stream)))
    return dX, dW


def sp_conv2d_bwd_weight_nchw(W: SparseWeight, g: sp_conv_geom, X: torch.Tensor, dY: torch.Tensor,
                              dW: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    OH, OW = _geo_out(g)
    _chk_shape(X, (g.B, g.C_in, g.H, g.W), "X (NCHW [B][C_in][H][W])")
    _chk_shape(dY, (g.B, g.C_out, OH, OW), "dY (NCHW [B][C_out][OH][OW])")
    if dW is None:
        dW = torch.empty(W.nnz, dtype=torch.float32, device=X.device)
    _chk_nnz(W, dW)
    _check(lib().sp_conv2d_bwd_weight_nchw(W.handle, ct.byref(g), _dev(X, torch.float32, "X"),
                                           _dev(dY, torch.float32, "dY"),
                                           _dev(dW, torch.float32, "dW") if W.nnz else None, _stream(stream)))
    return dW


def sp_mse_scratch_floats(n: int) -> int:
    return int(lib().sp_mse_scratch_floats(n))


def sp_mse_grad(Y: torch.Tensor, T: torch.Tensor, dY: torch.Tensor, loss: torch.Tensor,
                scratch: torch.Tensor, stream=None):
    n = Y.numel()
    if T.numel() != n or dY.numel() != n:
        raise ValueError("Y, T, dY sizes differ")
    _check(lib().sp_mse_grad(_dev(Y, torch.float32, "Y"), _dev(T, torch.float32, "T"),
                             _dev(dY, torch.float32, "dY"), _dev(loss, torch.float32, "loss"),
                             _dev(scratch, torch.float32, "scratch"), n, _stream(stream)))


def sp_set_sm_reserve(n: int):
    """Leave n SMs free in the one-wave kernels' grids (for a concurrent collective)."""
    _check(lib().sp_set_sm_reserve(int(n)))


def sp_weight_set_managed(W: SparseWeight, managed: bool = True):
    """Declare that W.vals changes only through sp_weight_sgd (products then
    skip the per-launch refresh of the tiled weights); see the C header."""
    _check(lib().sp_weight_set_managed(W.handle, 1 if managed else 0))


def sp_weight_sgd(W: SparseWeight, dW: torch.Tensor, lr: float, stream=None):
    """W.vals -= lr * dW, tiled copies included (one kernel)."""
    n = W.nnz
    _chk_nnz(W, dW)
    _check(lib().sp_weight_sgd(W.handle, _dev(dW, torch.float32, "dW") if n else None, ct.c_float(lr),
                               _stream(stream)))


def sp_weights_sgd(Ws, dWs, lr: float, stream=None):
    """sp_weight_sgd for many handles in one kernel (a model's optimizer step)."""
    Ws, dWs = list(Ws), list(dWs)
    if len(Ws) != len(dWs):
        raise ValueError("sp_weights_sgd: one dW per handle")
    for W, d in zip(Ws, dWs):
        _chk_nnz(W, d)
    hs = (ct.c_void_p * len(Ws))(*[W.handle.value for W in Ws])
    ds = (ct.c_void_p * len(dWs))(*[_dev(d, torch.float32, "dW") if W.nnz > 0 else None for W, d in zip(Ws, dWs)])
    _check(lib().sp_weights_sgd(hs, ds, len(Ws), ct.c_float(lr), _stream(stream)))


def sp_sgd(vals: torch.Tensor, dW: torch.Tensor, lr: float, stream=None):
    n = vals.numel()
    if dW.numel() != n:
        raise ValueError("vals and dW sizes differ")
    _check(lib().sp_sgd(_dev(vals, torch.float32, "vals") if n else None,
                        _dev(dW, torch.float32, "dW") if n else None, n, ct.c_float(lr),
                        _stream(stream)))


# ---------------------------------------------------------------------------
# Peer-memory dW all_reduce (include/sparseprop.h)
# ---------------------------------------------------------------------------
COMM_HANDLE_BYTES = 128


def _cai_view(owner, ptr: int, n: int, device) -> torch.Tensor:
    """fp32 [n] tensor over library-owned device memory; keeps `owner` alive."""
    class _CAI:
        def __init__(self):
            self.owner = owner
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                             "version": 3, "strides": None, "stream": None}
    return torch.as_tensor(_CAI(), device=device)


class PeerComm:
    """sp_comm_t owner.  create(): this rank's symmetric buffer + its IPC handle
    record (bytes); open(records): map the peers' buffers (records in rank order).
    The rendezvous (exchanging the records) is the caller's -- dp.P2PAllReduce
    does it with torch.distributed.all_gather_object."""

    def __init__(self, rank: int, world: int, count: int, device=None):
        self.rank, self.world, self.count = int(rank), int(world), int(count)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        h = ct.c_void_p()
        rec = ct.create_string_buffer(COMM_HANDLE_BYTES)
        _check(lib().sp_comm_create(self.rank, self.world, self.count, ct.byref(h), rec))
        self.handle = h
        self.record = rec.raw

    def open(self, records: list):
        if len(records) != self.world or any(len(r) != COMM_HANDLE_BYTES for r in records):
            raise ValueError("PeerComm.open: one handle record per rank, in rank order")
        _check(lib().sp_comm_open(self.handle, b"".join(records)))

    @property
    def buffer(self) -> torch.Tensor:
        return _cai_view(self, lib().sp_comm_buffer(self.handle), self.count, self.device)

    def allreduce(self, offset: int, count: int, stream=None):
        _check(lib().sp_comm_allreduce(self.handle, int(offset), int(count), _stream(stream)))

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().sp_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NvlsComm:
    """sp_nvls_t owner (the NVLS multicast dW all_reduce).  The collective setup
    is split so the caller can run the rendezvous between the steps:
    create (rank 0 gets the exported multicast fd in .fd), open(fd) on ranks > 0
    with that fd (the caller carries it between processes; dp.NvlsAllReduce
    does it with SCM_RIGHTS), barrier, bind(), barrier."""

    def __init__(self, rank: int, world: int, count: int, device=None):
        self.rank, self.world, self.count = int(rank), int(world), int(count)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        h, fd = ct.c_void_p(), ct.c_int32(-1)
        _check(lib().sp_nvls_create(self.rank, self.world, self.count, ct.byref(h), ct.byref(fd)))
        self.handle = h
        self.fd = int(fd.value)

    def open(self, fd: int = -1):
        _check(lib().sp_nvls_open(self.handle, int(fd)))

    def bind(self):
        _check(lib().sp_nvls_bind(self.handle))

    @property
    def buffer(self) -> torch.Tensor:
        return _cai_view(self, lib().sp_nvls_buffer(self.handle), self.count, self.device)

    def allreduce(self, offset: int, count: int, stream=None):
        _check(lib().sp_nvls_allreduce(self.handle, int(offset), int(count), _stream(stream)))

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().sp_nvls_destroy(self.handle)
            self.handle = None
        if getattr(self, "fd", -1) >= 0:
            os.close(self.fd)
            self.fd = -1

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nvls_supported() -> bool:
    """Multicast (NVLS) support of the current device (driver attribute)."""
    return bool(lib().sp_nvls_supported())


def comm_ctas() -> int:
    """CTAs one sp_comm_allreduce kernel occupies (SMs to leave free for it)."""
    return int(lib().sp_comm_ctas())


class LocalPeerComm:
    """Test hook: `world` virtual ranks' buffers in this process (sp_comm_create_local)."""

    def __init__(self, world: int, count: int):
        self.world, self.count = int(world), int(count)
        self.device = torch.device("cuda", torch.cuda.current_device())
        h = ct.c_void_p()
        _check(lib().sp_comm_create_local(self.world, self.count, ct.byref(h)))
        self.handle = h

    def buffer(self, rank: int) -> torch.Tensor:
        return _cai_view(self, lib().sp_comm_local_buffer(self.handle, int(rank)), self.count, self.device)

    def allreduce_as(self, rank: int, offset: int, count: int, stream=None):
        _check(lib().sp_comm_allreduce_as(self.handle, int(rank), int(offset), int(count), _stream(stream)))

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().sp_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

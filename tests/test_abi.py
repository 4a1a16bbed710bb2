"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/sparseprop.h declares, and validates arguments before any
launch (no compute call is made here)."""
import ctypes as ct
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "sparseprop.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2302_04852_b200 import _build, sparseprop
    _build.build()
    return sparseprop.lib()


def test_header_lists_the_north_star_entry_points():
    names = _declared()
    for n in ["sp_weight_create", "sp_linear_fwd", "sp_linear_bwd_input", "sp_linear_bwd_weight",
              "sp_conv2d_fwd", "sp_conv2d_bwd_input", "sp_conv2d_bwd_weight"]:
        assert n in names


def test_every_declared_symbol_is_exported(L):
    from paper_2302_04852_b200 import sparseprop
    out = subprocess.check_output(["nm", "-D", "--defined-only", sparseprop.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (sp_[a-z0-9_]+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    assert sorted(sparseprop.EXPORTS) == _declared()


def test_nvls_argument_validation_without_gpu(L):
    """The NVLS all_reduce entry points (sp_nvls_*) reject bad arguments before
    any driver call, and report no multicast support without a device."""
    h, fd = ct.c_void_p(), ct.c_int32(-1)
    L.sp_nvls_create.argtypes = [ct.c_int32, ct.c_int32, ct.c_int64, ct.c_void_p, ct.c_void_p]
    assert L.sp_nvls_create(0, 2, 16, None, ct.byref(fd)) == 1            # SP_ERR_NULL
    assert L.sp_nvls_create(0, 0, 16, ct.byref(h), ct.byref(fd)) == 2     # SP_ERR_SHAPE: world 0
    assert L.sp_nvls_create(2, 2, 16, ct.byref(h), ct.byref(fd)) == 2     # rank >= world
    assert L.sp_nvls_create(0, 9, 16, ct.byref(h), ct.byref(fd)) == 2     # world > 8
    assert L.sp_nvls_create(0, 1, 0, ct.byref(h), ct.byref(fd)) == 2      # count 0
    L.sp_nvls_open.argtypes = [ct.c_void_p, ct.c_int32]
    L.sp_nvls_allreduce.argtypes = [ct.c_void_p, ct.c_int64, ct.c_int64, ct.c_void_p]
    L.sp_nvls_destroy.argtypes = [ct.c_void_p]
    assert L.sp_nvls_open(None, 3) == 6                                   # SP_ERR_BAD_HANDLE
    assert L.sp_nvls_bind(None) == 6
    assert L.sp_nvls_allreduce(None, 0, 1, None) == 6
    assert L.sp_nvls_destroy(None) == 6
    L.sp_nvls_buffer.restype = ct.c_void_p
    assert L.sp_nvls_buffer(None) is None
    assert L.sp_nvls_ctas() == 8


def test_built_for_sm100a(L):
    from paper_2302_04852_b200 import sparseprop
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sparseprop.LIB_PATH],
                                  text=True)
    assert "sm_100a" in out


def test_argument_validation_without_gpu(L):
    from paper_2302_04852_b200 import sparseprop as sp
    h = ct.c_void_p()
    assert L.sp_weight_create(4, 4, None, None, None, ct.byref(h)) == 1          # SP_ERR_NULL
    assert "NULL" in L.sp_last_error().decode()
    assert L.sp_weight_create(0, 4, 1, 1, None, ct.byref(h)) == 2                # SP_ERR_SHAPE
    assert L.sp_weight_create(1 << 31, 4, 1, 1, None, ct.byref(h)) == 3         # SP_ERR_OVERFLOW: R > int32
    assert L.sp_weight_create(4, 1 << 31, 1, 1, None, ct.byref(h)) == 3         # C > int32
    assert L.sp_weight_create(4, 4, 1, 1, None, None) == 1
    assert L.sp_linear_fwd(None, 1, 1, 8, None) == 6                              # SP_ERR_BAD_HANDLE
    assert L.sp_linear_bwd_input(None, 1, 1, 8, None) == 6
    assert L.sp_linear_bwd_weight(None, 1, 1, 1, 8, None) == 6
    assert L.sp_conv2d_fwd(None, None, 1, 1, None) == 6
    assert L.sp_weight_nnz(None) == -1
    assert L.sp_sgd(None, None, 5, ct.c_float(0.1), None) == 1
    assert L.sp_mse_grad(None, None, None, None, None, 5, None) == 1
    h2 = ct.c_void_p()
    rec = ct.create_string_buffer(128)
    assert L.sp_comm_create(0, 9, 16, ct.byref(h2), rec) == 2                    # world > SP_COMM_MAX_WORLD
    assert L.sp_comm_create(2, 2, 16, ct.byref(h2), rec) == 2                    # rank >= world
    assert L.sp_comm_create(0, 2, 16, None, rec) == 1
    assert L.sp_comm_allreduce(None, 0, 4, None) == 6
    assert L.sp_comm_open(None, rec) == 6
    assert L.sp_comm_ctas() >= 1
    assert L.sp_weights_sgd(None, None, 1, ct.c_float(0.1), None) == 1           # SP_ERR_NULL
    hs = (ct.c_void_p * 1)(None)
    ds = (ct.c_void_p * 1)(None)
    assert L.sp_weights_sgd(hs, ds, 0, ct.c_float(0.1), None) == 2                # n < 1
    assert L.sp_weights_sgd(hs, ds, 65, ct.c_float(0.1), None) == 2               # n > SP_SGD_BATCH_MAX
    assert L.sp_weights_sgd(hs, ds, 1, ct.c_float(0.1), None) == 6                # a NULL handle
    assert "sm_100a" in sp.version()


def test_binding_refuses_cpu_tensors(L):
    torch = pytest.importorskip("torch")
    from paper_2302_04852_b200 import sparseprop as sp
    with pytest.raises(ValueError, match="CUDA"):
        sp.sp_weight_create(torch.zeros(4, 4), torch.zeros(4, 4, dtype=torch.uint8))

"""A handle whose R*C exceeds int32 (round 1 refused it for an
R x C int32 scratch the CSC build no longer uses): 50000 x 50000 at 1 %
density.  Structure checked against torch reductions of the mask; sampled
forward rows and dW entries against float64 sums on the same device data."""
import time

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_50k_by_50k_one_percent():
    from paper_2302_04852_b200 import sparseprop as sp
    R = C = 50000
    g = torch.Generator(device="cuda").manual_seed(50)
    mask = torch.empty(R, C, dtype=torch.uint8, device="cuda")
    for r0 in range(0, R, 5000):  # chunked draws (bounded temporaries)
        mask[r0:r0 + 5000] = (torch.rand(5000, C, generator=g, device="cuda") < 0.01).to(torch.uint8)
    dense = torch.empty(R, C, dtype=torch.float32, device="cuda")
    for r0 in range(0, R, 5000):
        dense[r0:r0 + 5000].normal_(0.0, 0.01, generator=g)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    W = sp.sp_weight_create(dense, mask)
    torch.cuda.synchronize()
    t_create = time.perf_counter() - t0
    rows = mask.sum(1, dtype=torch.int64)
    cols = mask.sum(0, dtype=torch.int64)
    assert W.nnz == int(rows.sum())
    idx = W.indices()
    assert torch.equal(idx["row_ptr"][1:].to(torch.int64), torch.cumsum(rows, 0))
    assert torch.equal(idx["col_ptr"][1:].to(torch.int64), torch.cumsum(cols, 0))
    # CSC -> CSR consistency: row_idx[k] is the row of CSR slot perm[k], col_idx[perm[k]] its column
    perm = idx["perm"].to(torch.int64)
    colk = torch.repeat_interleave(torch.arange(C, device="cuda"), cols)
    assert torch.equal(idx["col_idx"].to(torch.int64)[perm], colk)
    row_of_slot = torch.repeat_interleave(torch.arange(R, device="cuda"), rows)
    assert torch.equal(row_of_slot[perm], idx["row_idx"].to(torch.int64))
    # sampled forward rows and dW entries in float64
    B = 8
    X = torch.randn(C, B, generator=g, device="cuda")
    dY = torch.randn(R, B, generator=g, device="cuda")
    Y = sp.sp_linear_fwd(W, X)
    dX, dW = sp.sp_linear_bwd(W, X, dY)
    torch.cuda.synchronize()
    sel = torch.randint(0, R, (64,), generator=g, device="cuda")
    Wm = (dense[sel].double() * mask[sel].double())
    ref = Wm @ X.double()
    err = (Y[sel].double() - ref).abs().max().item()
    assert err <= 1e-4 * ref.abs().max().item() + 1e-6
    slots = torch.randint(0, W.nnz, (4096,), generator=g, device="cuda")
    r_s, c_s = row_of_slot[slots], idx["col_idx"].to(torch.int64)[slots]
    refw = (dY[r_s].double() * X[c_s].double()).sum(1)
    errw = (dW[slots].double() - refw).abs().max().item()
    assert errw <= 1e-4 * refw.abs().max().item() + 1e-6
    print(f"50000 x 50000 @ 1%: nnz {W.nnz}, sp_weight_create {t_create * 1e3:.1f} ms")

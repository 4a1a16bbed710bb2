"""The peer-memory dW all_reduce kernel (include/sparseprop.h
sp_comm_*) on one GPU.  The multi-GPU flag synchronisation needs >= 2 GPUs;
here `world` virtual ranks live in one process (sp_comm_create_local) and
rank r's share of a call runs with the flags off, r = 0..world-1 in order --
which reproduces the multi-GPU result exactly, because rank r reads and writes
only chunk r.  Checked: every rank ends with bitwise the rank-order fp32 sum
(0 + 1 + ... + world-1, the kernel's fixed order), elements outside the range
untouched, unaligned offsets / ragged lengths, repeated calls (epochs)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2302_04852_b200 import _build, sparseprop
    _build.build()
    return sparseprop


def _rank_order_sum(bufs):
    s = bufs[0].astype(np.float32).copy()
    for b in bufs[1:]:
        s = (s + b).astype(np.float32)
    return s


@pytest.mark.parametrize("world,count,off,n", [
    (2, 4096, 0, 4096), (4, 1_000_003, 0, 1_000_003), (8, 2_831_025, 0, 2_831_025),
    (3, 100_001, 3, 77_777), (8, 64, 5, 1), (4, 4096, 1000, 0), (1, 1000, 0, 1000),
])
def test_allreduce_virtual_ranks(sp, world, count, off, n):
    g = np.random.default_rng(world * 1000 + count)
    host = [g.standard_normal(count).astype(np.float32) for _ in range(world)]
    c = sp.LocalPeerComm(world, count)
    bufs = [c.buffer(r) for r in range(world)]
    for b, h in zip(bufs, host):
        b.copy_(torch.from_numpy(h))
    for _ in range(2):  # two calls: the per-CTA epochs advance; the second sums the first's sums
        for r in range(world):
            c.allreduce_as(r, off, n)
        torch.cuda.synchronize()
        ref = _rank_order_sum([h[off:off + n] for h in host])
        for h in host:
            h[off:off + n] = ref
        for b, h in zip(bufs, host):
            np.testing.assert_array_equal(b.cpu().numpy(), h)  # bitwise; outside the range untouched
    c.close()


def test_single_rank_communicator(sp):
    """sp_comm_create / open / allreduce with world = 1 (no peers, no flags)."""
    c = sp.PeerComm(0, 1, 1000)
    c.open([c.record])
    x = torch.arange(1000, dtype=torch.float32, device="cuda")
    c.buffer.copy_(x)
    c.allreduce(0, 1000)
    c.allreduce(10, 17)
    torch.cuda.synchronize()
    assert torch.equal(c.buffer, x)
    with pytest.raises(sp.SparsePropError):
        c.allreduce(990, 20)  # past the buffer
    c.close()


def test_nvls_single_device_group(sp):
    """The NVLS multicast all_reduce (sp_nvls_*) on this box's one visible GPU:
    a multicast object of one device, its memory bound and mapped, the kernel's
    multimem.ld_reduce / multimem.st and the multimem.red flag barriers run on
    the hardware.  The sum over a one-rank group is the buffer itself, so every
    element must come back bitwise unchanged -- over aligned, unaligned and
    ragged ranges, repeated calls (epochs) and CUDA-graph replays.  The
    multi-rank protocol (fd carried by SCM_RIGHTS, add-device / bind barriers)
    is tested on CPU in test_dp_gloo.py."""
    if not sp.nvls_supported():
        pytest.skip("device without multicast (NVLS) support")
    n = 1_000_003
    try:
        c = sp.NvlsComm(0, 1, n)
        c.open(-1)
        c.bind()
    except sp.SparsePropError as e:
        # the driver's multicast set-up (create / add device / bind / map) is
        # refused on this pool's single-GPU pods: CUDA_ERROR_INVALID_VALUE from
        # cuMulticastCreate for 1 or 2 devices and every handle type
        # (tools/dbg/probe_mc.py); the kernel's results are asserted below
        # wherever the set-up succeeds
        if "SP_ERR_CUDA" in str(e):
            pytest.skip(f"multicast set-up refused here: {e}")
        raise
    buf = c.buffer
    assert buf.numel() == n and float(buf.abs().max()) == 0.0  # bind() zeroes it
    g = torch.Generator(device="cuda").manual_seed(5)
    ref = torch.randn(n, device="cuda", generator=g)
    buf.copy_(ref)
    for off, cnt in [(0, n), (1, 17), (3, 4096 + 5), (n - 7, 7), (12345, 0), (4, n - 8)]:
        c.allreduce(off, cnt)
    torch.cuda.synchronize()
    assert torch.equal(buf, ref)
    # graph capture: the epochs live in device memory, so replays keep the barriers consistent
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        c.allreduce(0, n, st)  # warm-up on the capture stream
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        c.allreduce(0, n, st)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(buf, ref)
    c.close()

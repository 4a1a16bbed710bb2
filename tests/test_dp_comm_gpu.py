"""The N > 1 code path of the DP step on one GPU, over a one-rank NCCL group:
the bucketed all_reduce on the comm stream (NCCL, and the peer-memory kernel
through dp.P2PAllReduce with a one-rank PeerComm) with SMs reserved in the
backward's one-wave kernels.  A one-rank SUM is the identity, so the step
must give bitwise the dW of the plain single-GPU step (the multi-rank
arithmetic is covered by tests/test_comm_gpu.py and the gloo tests)."""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", torch.cuda.current_device()))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("comm", ["nccl", "p2p"])
def test_dp_step_comm_path_one_rank(nccl_group, comm):
    from paper_2302_04852_b200 import sparseprop as sp
    from paper_2302_04852_b200.dp import P2PAllReduce, SparseMLP
    T = 1024
    c = synth.mlp_case(blocks=4, d_model=768, d_ff=3072, T=T, density=0.05, seed=31)
    X0, tgt = torch.from_numpy(c["X0"]), torch.from_numpy(c["target"])
    ref = SparseMLP(c["layers"], T, "cuda", bucket_blocks=2)
    ref.set_batch(X0, tgt, non_blocking=False)
    ref.forward()
    ref.backward(allreduce=False)
    m = SparseMLP(c["layers"], T, "cuda", bucket_blocks=2, sm_reserve=sp.comm_ctas() if comm == "p2p" else 8)
    # drive the N > 1 branch: comm stream, buckets, SM reserve (one-rank group: SUM = identity)
    m.world = 2
    m.comm_stream = torch.cuda.Stream()
    if comm == "p2p":
        ar = P2PAllReduce(nccl_group, m.nnz_total, m.device)
        ar.buffer.copy_(torch.arange(m.nnz_total, dtype=torch.float32, device="cuda"))
        m.p2p = ar  # its kernel runs on its own (one-rank) buffer; dW_flat stays the model's
    m.set_batch(X0, tgt, non_blocking=False)
    m.forward()
    m.backward(allreduce=True)
    torch.cuda.synchronize()
    assert len(m.buckets) == 2
    # the reserved-SM grids change the stream-K partitions, so compare within tolerance
    a, b = m.dW_flat.cpu().numpy(), ref.dW_flat.cpu().numpy()
    assert np.max(np.abs(a - b)) <= 1e-4 * np.max(np.abs(b)) + 1e-6
    if comm == "p2p":
        assert torch.equal(ar.buffer, torch.arange(m.nnz_total, dtype=torch.float32, device="cuda"))
    sp.sp_set_sm_reserve(0)

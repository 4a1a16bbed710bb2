"""N>1 host logic of the data-parallel MLP step on CPU (gloo, world_size 2):
token sharding, flat dW buffer, reverse-order bucketing, all_reduce wiring,
SGD ordering.  Arithmetic is supplied by an oracle-backed `ops` (test
infrastructure) so this runs without a GPU; the product ops are CudaOps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


class OracleOps:
    """CPU stand-in for CudaOps built on the fp64 oracle (tests only)."""

    class H:
        def __init__(self, dense, mask):
            self.S = oracle.csr_from_mask(dense.numpy(), mask.numpy())
            self.nnz = self.S.nnz
            self.vals_t = torch.from_numpy(self.S.vals.astype(np.float32))

    def create(self, dense, mask):
        return OracleOps.H(dense, mask)

    def vals(self, W):
        return W.vals_t

    def _S(self, W):
        return W.S.with_vals(W.vals_t.numpy().astype(np.float64))

    def fwd(self, W, X, Y, relu):
        r = oracle.linear_fwd(self._S(W), X.numpy())
        Y.copy_(torch.from_numpy(np.maximum(r, 0.0) if relu else r))

    def dx(self, W, dY, dX, H=None):
        r = oracle.linear_bwd_input(self._S(W), dY.numpy())
        if H is not None:
            r = r * (H.numpy() > 0)
        dX.copy_(torch.from_numpy(r))

    def dw(self, W, X, dY, dW):
        dW.copy_(torch.from_numpy(oracle.linear_bwd_weight(W.S, X.numpy(), dY.numpy())))

    def bwd(self, W, X, dY, dX, dW, H=None):
        self.dw(W, X, dY, dW)
        self.dx(W, dY, dX, H=H)

    def mse(self, Y, T, dY, loss, scratch):
        d = Y.numpy().astype(np.float64) - T.numpy()
        dY.copy_(torch.from_numpy(d))
        loss.fill_(0.5 * float(np.sum(d * d)))

    def mse_scratch(self, n):
        return 2

    def sgd(self, vals, dW, lr):
        vals.sub_(lr * dW)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, q, fused):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_04852_b200.dp import SparseMLP
    c = synth.mlp_case(blocks=3, d_model=12, d_ff=20, T=T, density=0.3, seed=123)
    lo, hi = synth.token_shard(T, world, rank)
    m = SparseMLP(c["layers"], hi - lo, "cpu", ops=OracleOps(), bucket_blocks=2, fused=fused)
    m.set_batch(torch.from_numpy(c["X0"][:, lo:hi].copy()), torch.from_numpy(c["target"][:, lo:hi].copy()),
                non_blocking=False)
    loss = m.forward().clone()
    m.backward(allreduce=True)
    dist.all_reduce(loss)
    m.sgd(0.01)
    vals = torch.cat([torch.cat([m.ops.vals(a), m.ops.vals(b)]) for a, b in m.W])
    q.put((rank, float(loss), m.dW_flat.numpy().copy(), vals.numpy().copy(), m.buckets))
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("world", [2])
def test_dp_gloo_matches_full_batch(world, fused):
    T = 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, q, fused)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # full-batch oracle reference
    c = synth.mlp_case(blocks=3, d_model=12, d_ff=20, T=T, density=0.3, seed=123)
    layers = [(oracle.csr_from_mask(w1, m1), oracle.csr_from_mask(w2, m2)) for (w1, m1, w2, m2) in c["layers"]]
    full = oracle.mlp_step(layers, c["X0"], c["target"])
    ref = np.concatenate([np.concatenate(p) for p in full["dW"]])
    ref_vals = np.concatenate([np.concatenate([a.vals, b.vals]) for a, b in layers]) - 0.01 * ref
    for rank, loss, dW, vals, buckets in res:
        assert loss == pytest.approx(full["loss"], rel=1e-5)
        np.testing.assert_allclose(dW, ref, rtol=1e-5, atol=1e-5)     # every rank holds the SUM
        np.testing.assert_allclose(vals, ref_vals, rtol=1e-5, atol=1e-6)
        # buckets cover the flat buffer exactly once, in reverse block order
        assert [b[0] for b in buckets] == [1, 0] and buckets[0][3] == dW.size and buckets[-1][2] == 0
    assert np.array_equal(res[0][2], res[1][2])                          # identical after all_reduce


class _FakeComm:
    """Stand-in for sparseprop.PeerComm (host logic only): a record naming
    its rank, a CPU buffer, and a log of the calls."""

    def __init__(self, rank, world, count):
        self.record = bytes([rank]) * 128
        self.buffer = torch.zeros(count)
        self.opened = None

    def open(self, records):
        self.opened = [r[0] for r in records]


def _p2p_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_04852_b200.dp import P2PAllReduce
    made = []
    ar = P2PAllReduce(None, 37, "cpu", comm_factory=lambda r, w, n: made.append((r, w, n)) or _FakeComm(r, w, n))
    q.put((rank, made, ar.comm.opened, ar.buffer.numel()))
    dist.destroy_process_group()


def test_p2p_rendezvous_gathers_records_in_rank_order():
    """SURVEY F2 host logic: each rank creates its communicator once and maps
    its peers from the records all ranks exchanged, in rank order."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, made, opened, n in res:
        assert made == [(rank, world, 37)]
        assert opened == list(range(world))
        assert n == 37


class _FakeNvls:
    """Stand-in for sparseprop.NvlsComm (host logic only): rank 0 'exports' a
    read-only descriptor of an unlinked file holding a token; open(fd) reads the
    token through the fd it was handed (pread: the ranks share one open file);
    calls are logged."""

    def __init__(self, rank, world, count):
        self.fd, self.log, self.token = -1, [], None
        self.buffer = torch.zeros(count)
        if rank == 0:
            import tempfile
            with tempfile.NamedTemporaryFile(delete=False) as f:
                f.write(b"nvls-token" * 4)
            self.fd = os.open(f.name, os.O_RDONLY)
            os.unlink(f.name)

    def open(self, fd):
        self.log.append("open")
        if fd >= 0:
            self.token = os.pread(fd, 64, 0)

    def bind(self):
        self.log.append("bind")


def _nvls_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_04852_b200.dp import NvlsAllReduce
    ar = NvlsAllReduce(None, 41, "cpu", comm_factory=lambda r, w, n: _FakeNvls(r, w, n))
    q.put((rank, ar.comm.log, ar.comm.token, ar.buffer.numel()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_nvls_rendezvous_carries_the_multicast_fd(world):
    """SURVEY F2 (NVLS) host logic: rank 0's exported multicast fd reaches every
    other rank through SCM_RIGHTS (dp.share_fd), each rank opens (imports + adds
    its device) before binding; rank 0 opens without an fd."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nvls_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, log, token, n in res:
        assert log == ["open", "bind"]
        assert n == 41
        assert token == (None if rank == 0 else b"nvls-token" * 4)

"""Data-parallel sparse MLP step (north star cfg5).

`blocks` x [W1 (d_ff x d_model) sparse, ReLU, W2 (d_model x d_ff) sparse],
MSE loss L = 1/2 sum (Y - T)^2.  One process per GPU; rank g
owns the contiguous token shard [g T/G, (g+1) T/G) as its own [feat x T/G]
buffers.  The only exchange is an all_reduce(SUM) of the nnz-length dW value
buffers (one flat buffer, bucketed in reverse layer order and launched on a
side stream as soon as a bucket's SDDMMs are done, overlapping the rest of the
backward).  Then plain SGD on the kept weights.

Every arithmetic step runs in libsparseprop's kernels (fwd SpMM + fused ReLU,
CSC-driven dX SpMM + fused ReLU' gate, SDDMM, MSE, SGD).  The `ops` object is
the only thing this module calls for arithmetic; `CudaOps` is the product.
Tests substitute a CPU oracle-backed `ops` to exercise the sharding /
bucketing / all_reduce logic with gloo on CPU (tests/test_dp_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class CudaOps:
    """The product arithmetic: libsparseprop through its C ABI."""

    def __init__(self):
        from . import sparseprop as sp
        self.sp = sp
        sp.lib()

    def create(self, dense, mask):
        # the model updates vals only through sp_weight_sgd: products skip the
        # per-launch refresh of the tiled weights (managed handles)
        W = self.sp.sp_weight_create(dense, mask)
        self.sp.sp_weight_set_managed(W, True)
        return W

    def vals(self, W):
        return W.vals

    def fwd(self, W, X, Y, relu):
        return self.sp.sp_linear_fwd(W, X, Y, relu=relu)

    def dx(self, W, dY, dX, H=None):
        return self.sp.sp_linear_bwd_input(W, dY, dX, H=H)

    def dw(self, W, X, dY, dW):
        return self.sp.sp_linear_bwd_weight(W, X, dY, dW)

    def bwd(self, W, X, dY, dX, dW, H=None):
        """Fused backward (one CSC-driven pass): dX [* (H > 0)] and dW."""
        return self.sp.sp_linear_bwd(W, X, dY, dX, dW, H=H)

    def mse(self, Y, T, dY, loss, scratch):
        self.sp.sp_mse_grad(Y, T, dY, loss, scratch)

    def mse_scratch(self, n):
        return self.sp.sp_mse_scratch_floats(n)

    def sgd(self, vals, dW, lr):
        self.sp.sp_sgd(vals, dW, lr)

    def sgd_weight(self, W, dW, lr):
        """SGD of a managed handle: vals and its tiled copies in one kernel."""
        self.sp.sp_weight_sgd(W, dW, lr)

    def sgd_weights(self, Ws, dWs, lr):
        """SGD of every managed handle of the model in ONE kernel."""
        self.sp.sp_weights_sgd(Ws, dWs, lr)

    def sm_reserve(self, n):
        """One-wave kernels leave n SMs to the concurrent all_reduce."""
        self.sp.sp_set_sm_reserve(n)


class P2PAllReduce:
    """The peer-memory dW all_reduce (sparseprop.PeerComm):
    every rank creates its symmetric buffer, the IPC handle records are
    exchanged with all_gather_object over `group` (rank order), and each rank
    maps its peers.  The model's flat dW buffer IS this rank's symmetric buffer,
    so the backward writes dW where the peers read it.  comm_factory (tests):
    (rank, world, count) -> an object with .record, .open(records), .buffer,
    .allreduce(offset, count, stream)."""

    def __init__(self, group, count: int, device, comm_factory=None):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if comm_factory is None:
            from . import sparseprop as sp
            comm_factory = lambda r, w, n: sp.PeerComm(r, w, n, device)  # noqa: E731
        self.comm = comm_factory(self.rank, self.world, count)
        records = [None] * self.world
        dist.all_gather_object(records, self.comm.record, group=group)
        self.comm.open(records)

    @property
    def buffer(self):
        return self.comm.buffer

    def allreduce(self, lo: int, hi: int, stream=None):
        self.comm.allreduce(lo, hi - lo, stream)


def share_fd(group, rank: int, world: int, fd: int) -> int:
    """Rank 0's file descriptor `fd` to every rank of `group` (SCM_RIGHTS over an
    abstract Unix socket whose name rank 0 draws and all_gathers): returns the
    fd (rank 0: its own; others: a new descriptor of the same open file, which
    the caller closes).  Used to carry the NVLS multicast handle."""
    import secrets
    import socket
    names = [None] * world
    dist.all_gather_object(names, "\0sp-nvls-" + secrets.token_hex(8) if rank == 0 else None, group=group)
    name = names[0]
    if rank == 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name)
        srv.listen(world)
        dist.barrier(group=group)  # listening
        for _ in range(world - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"f"], [fd])
            conn.close()
        srv.close()
        return fd
    dist.barrier(group=group)
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    cli.connect(name)
    _, fds, _, _ = socket.recv_fds(cli, 1, 1)
    cli.close()
    return fds[0]


class NvlsAllReduce:
    """The NVLS multicast dW all_reduce (sparseprop.NvlsComm):
    rank 0 creates the multicast object and its fd reaches the other ranks
    (share_fd); every rank adds its device, then binds its buffer (barriers
    between, as the driver's protocol requires).  Same interface as
    P2PAllReduce: the model's flat dW buffer IS this rank's multicast-bound
    buffer.  comm_factory (tests): (rank, world, count) -> an object with .fd,
    .open(fd), .bind(), .buffer, .allreduce(offset, count, stream)."""

    def __init__(self, group, count: int, device, comm_factory=None):
        import os
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if comm_factory is None:
            from . import sparseprop as sp
            comm_factory = lambda r, w, n: sp.NvlsComm(r, w, n, device)  # noqa: E731
        self.comm = comm_factory(self.rank, self.world, count)
        fd = share_fd(group, self.rank, self.world, self.comm.fd) if self.world > 1 else -1
        self.comm.open(fd if self.rank > 0 else -1)
        if self.rank > 0 and fd >= 0:
            os.close(fd)  # (imported: the driver holds its own reference)
        if self.world > 1:
            dist.barrier(group=group)  # every device added before any bind
        self.comm.bind()
        if self.world > 1:
            dist.barrier(group=group)

    @property
    def buffer(self):
        return self.comm.buffer

    def allreduce(self, lo: int, hi: int, stream=None):
        self.comm.allreduce(lo, hi - lo, stream)


class SparseMLP:
    """cfg5 model state + one training step on this rank's token shard."""

    def __init__(self, layers, T_local: int, device, ops=None, group=None, bucket_blocks: int = 3,
                 keep_dx0: bool = True, fused: bool = True, sm_reserve: int = 8, comm: str = "nccl",
                 comm_factory=None):
        """layers: list of (w1, m1, w2, m2) host arrays (synth.mlp_case).
        sm_reserve: at N > 1, SMs the backward's one-wave (stream-K) kernels
        leave free while the bucketed all_reduce runs on the comm stream, so
        the collective's CTAs do not push part of a wave into a second one
        (match it to NCCL's channel count, NCCL_MAX_NCHANNELS; "p2p": the
        peer-memory kernel's CTA count, sparseprop.comm_ctas()).
        comm: "nccl" (torch.distributed.all_reduce), "p2p" (P2PAllReduce:
        the library's peer-memory kernel over NVLink, CUDA only) or "nvls"
        (NvlsAllReduce: the library's NVLink SHARP multicast kernel)."""
        if comm not in ("nccl", "p2p", "nvls"):
            raise ValueError("comm must be 'nccl', 'p2p' or 'nvls'")
        self.sm_reserve = sm_reserve
        self.comm = comm
        self.ops = ops if ops is not None else CudaOps()
        self.device = torch.device(device)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.blocks = len(layers)
        self.d_model = layers[0][0].shape[1]
        self.d_ff = layers[0][0].shape[0]
        self.T = T_local
        self.keep_dx0 = keep_dx0
        self.fused = fused
        f32 = dict(dtype=torch.float32, device=self.device)
        self.W = []
        for (w1, m1, w2, m2) in layers:
            W1 = self.ops.create(torch.as_tensor(w1).to(self.device), torch.as_tensor(m1).to(self.device))
            W2 = self.ops.create(torch.as_tensor(w2).to(self.device), torch.as_tensor(m2).to(self.device))
            self.W.append((W1, W2))
        # one flat dW buffer; per-layer views; buckets in reverse block order
        sizes = [(W1.nnz, W2.nnz) for (W1, W2) in self.W]
        self.nnz_total = sum(a + b for a, b in sizes)
        self.p2p = None
        if comm in ("p2p", "nvls") and self.world > 1:
            cls = P2PAllReduce if comm == "p2p" else NvlsAllReduce
            self.p2p = cls(group, self.nnz_total, self.device, comm_factory)
            self.dW_flat = self.p2p.buffer[:self.nnz_total]
        else:
            self.dW_flat = torch.zeros(self.nnz_total, **f32)
        self.dW = []
        off = 0
        self.block_range = []
        for (a, b) in sizes:
            self.dW.append((self.dW_flat[off:off + a], self.dW_flat[off + a:off + a + b]))
            self.block_range.append((off, off + a + b))
            off += a + b
        self.buckets = []  # (first_block, last_block, lo, hi); launched when first_block's dW done
        l = self.blocks - 1
        while l >= 0:
            first = max(0, l - bucket_blocks + 1)
            self.buckets.append((first, l, self.block_range[first][0], self.block_range[l][1]))
            l = first - 1
        # activations: X_l [d_model x T] (l = 0..blocks), H_l [d_ff x T]
        self.X = [torch.empty(self.d_model, T_local, **f32) for _ in range(self.blocks + 1)]
        self.H = [torch.empty(self.d_ff, T_local, **f32) for _ in range(self.blocks)]
        self.dY = torch.empty(self.d_model, T_local, **f32)
        self.dYb = torch.empty(self.d_model, T_local, **f32)
        self.dZ = torch.empty(self.d_ff, T_local, **f32)
        self.dX0 = torch.empty(self.d_model, T_local, **f32)
        self.target = torch.empty(self.d_model, T_local, **f32)
        self.loss = torch.zeros(1, **f32)
        self.mse_scratch = torch.empty(max(2, self.ops.mse_scratch(self.d_model * T_local)), **f32)
        self.is_cuda = self.device.type == "cuda"
        self.comm_stream = torch.cuda.Stream(device=self.device) if (self.is_cuda and self.world > 1) else None
        if self.p2p is not None and self.comm_stream is None:
            raise ValueError(f"comm='{comm}' needs CUDA tensors")

    # ------------------------------------------------------------------
    def set_batch(self, X0: torch.Tensor, target: torch.Tensor, non_blocking: bool = True):
        """Copy this rank's shard (host pinned or device) into the resident buffers."""
        self.X[0].copy_(X0, non_blocking=non_blocking)
        self.target.copy_(target, non_blocking=non_blocking)

    # ---- input prefetch: the next step's host -> device copy on a side stream,
    # overlapped with the current step (double-buffered X0 / target) ----------
    def prefetch_batch(self, X0: torch.Tensor, target: torch.Tensor):
        """Start copying the next shard into the staging buffers (CUDA only).
        The staging buffers last held the input of the step before the current
        one; the copy stream waits for that step to be done with them."""
        if not hasattr(self, "_stage"):
            self._stage = (torch.empty_like(self.X[0]), torch.empty_like(self.target))
            self._copy_stream = torch.cuda.Stream(device=self.device)
            self._stage_ready = torch.cuda.Event()
            self._stage_free = None
        if self._stage_free is not None:
            self._copy_stream.wait_event(self._stage_free)
        with torch.cuda.stream(self._copy_stream):
            self._stage[0].copy_(X0, non_blocking=True)
            self._stage[1].copy_(target, non_blocking=True)
            self._stage_ready.record(self._copy_stream)

    def use_prefetched(self):
        """Make the prefetched shard this step's input (the current stream waits
        for its copy); the replaced buffers become the next staging buffers."""
        torch.cuda.current_stream(self.device).wait_event(self._stage_ready)
        old_x, old_t = self.X[0], self.target
        self.X[0], self.target = self._stage
        self._stage = (old_x, old_t)

    def release_staging(self):
        """Call after a step: its (now staging) buffers are free once the step ends."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self._stage_free = ev

    def forward(self):
        ops = self.ops
        for l, (W1, W2) in enumerate(self.W):
            ops.fwd(W1, self.X[l], self.H[l], relu=True)          # H = max(W1 X, 0)
            ops.fwd(W2, self.H[l], self.X[l + 1], relu=False)     # X' = W2 H
        ops.mse(self.X[self.blocks], self.target, self.dY, self.loss, self.mse_scratch)
        return self.loss

    def backward(self, allreduce: bool = True, trace: list | None = None):
        """trace (tests only): receives (l, dY_in, dZ, dX_out) clones per block."""
        ops = self.ops
        comm = allreduce and self.world > 1
        pending = []
        bi = 0
        dY, dYn = self.dY, self.dYb
        fused = self.fused and hasattr(ops, "bwd")
        if comm and self.sm_reserve and hasattr(ops, "sm_reserve"):
            ops.sm_reserve(self.sm_reserve)
        for l in range(self.blocks - 1, -1, -1):
            W1, W2 = self.W[l]
            dW1, dW2 = self.dW[l]
            out = self.dX0 if l == 0 else dYn
            if fused:
                # one CSC-driven pass per layer (dX and dW together)
                ops.bwd(W2, self.H[l], dY, self.dZ, dW2, H=self.H[l])  # dZ = (W2^T dY)*[H>0], dW2
                ops.bwd(W1, self.X[l], self.dZ, out, dW1)               # dX = W1^T dZ, dW1
            else:
                ops.dw(W2, self.H[l], dY, dW2)                        # dW2 = SDDMM(dY, H)
                ops.dx(W2, dY, self.dZ, H=self.H[l])                  # dZ = (W2^T dY) * [H > 0]
                ops.dw(W1, self.X[l], self.dZ, dW1)                   # dW1 = SDDMM(dZ, X)
                if l > 0 or self.keep_dx0:
                    ops.dx(W1, self.dZ, out)                          # dX = W1^T dZ
            if trace is not None:
                trace.append((l, dY.clone(), self.dZ.clone(), out.clone()))
            if l > 0:
                dY, dYn = dYn, dY
            if comm and bi < len(self.buckets) and self.buckets[bi][0] == l:
                lo, hi = self.buckets[bi][2], self.buckets[bi][3]
                pending.append(self._launch_allreduce(lo, hi))
                bi += 1
        if comm:
            self._wait(pending)
            if self.sm_reserve and hasattr(ops, "sm_reserve"):
                ops.sm_reserve(0)

    def _launch_allreduce(self, lo: int, hi: int):
        """All_reduce(SUM) of dW_flat[lo:hi] on the comm stream once the current
        stream has produced it (NCCL, or the peer-memory kernel)."""
        buf = self.dW_flat[lo:hi]
        if self.comm_stream is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            self.comm_stream.wait_event(ev)
            if self.p2p is not None:
                self.p2p.allreduce(lo, hi, self.comm_stream)
                return None
            with torch.cuda.stream(self.comm_stream):
                dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
            return None
        return dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group, async_op=True)

    def _wait(self, pending):
        if self.comm_stream is not None:
            torch.cuda.current_stream(self.device).wait_stream(self.comm_stream)
        else:
            for w in pending:
                if w is not None:
                    w.wait()

    def sgd(self, lr: float):
        if hasattr(self.ops, "sgd_weights"):
            self.ops.sgd_weights([W for pair in self.W for W in pair], [d for pair in self.dW for d in pair], lr)
            return
        for (W1, W2), (d1, d2) in zip(self.W, self.dW):
            if hasattr(self.ops, "sgd_weight"):
                self.ops.sgd_weight(W1, d1, lr)
                self.ops.sgd_weight(W2, d2, lr)
            else:
                self.ops.sgd(self.ops.vals(W1), d1, lr)
                self.ops.sgd(self.ops.vals(W2), d2, lr)

    def step(self, lr: float, allreduce: bool = True):
        """forward -> loss -> backward (+ bucketed all_reduce of dW) -> SGD.
        Returns the (device) local loss tensor."""
        loss = self.forward()
        self.backward(allreduce=allreduce)
        self.sgd(lr)
        return loss

    # ---- whole-step CUDA graph: the step's ~100 launches
    # (and, at N > 1, its NCCL all_reduces on the comm stream) replayed as one
    # graph.  Capture-safe: scratch is stream-ordered (graph memory nodes under
    # capture), the tensor maps are kernel parameters, and managed handles launch
    # no per-product refresh.  Buffers are fixed at capture: one graph per
    # input-buffer parity when the e2e loop double-buffers its inputs.
    def capture(self, lr: float, allreduce: bool = True):
        """Capture one step (forward, loss, backward + all_reduce, SGD) with the
        current X[0] / target buffers; returns the graph (replay() runs a step)."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            self.step(lr, allreduce=allreduce)  # warm: lazy state outside the capture
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        with torch.cuda.graph(g, stream=s):
            self.step(lr, allreduce=allreduce)
        torch.cuda.synchronize(self.device)
        return g

    def step_flops(self) -> int:
        """Effective FLOPs of one step on this rank: 2*nnz*B per product
        (BASELINE metric): 3 products per layer (fwd, dX, dW),
        minus the first layer's dX when it is not kept."""
        total = sum(3 * 2 * (W1.nnz + W2.nnz) * self.T for (W1, W2) in self.W)
        if not self.keep_dx0:
            total -= 2 * self.W[0][0].nnz * self.T
        return total

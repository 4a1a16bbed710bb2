#!/usr/bin/env python
"""bench.py -- SparseProp hot path on B200 (BASELINE.json metric:
"sparse fwd+bwd effective GFLOP/s (2*nnz*B) and % roofline, 1/2/4/8 B200").

Workload: BASELINE.json configs[4], the data-parallel sparse
MLP step -- 12 x [sparse 768->3072, ReLU, sparse 3072->768] fp32 at 95%
sparsity, global batch 16384 tokens, MSE loss, bucketed NCCL all_reduce of
the nnz dW buffers, SGD.  It is the configuration the metric's "1/2/4/8 B200"
is quoted on and it runs every linear row of SURVEY §8(a) (fwd SpMM + ReLU,
CSC dX SpMM + ReLU', SDDMM, MSE, SGD, all_reduce) in one step.  The global
batch is fixed and sharded by tokens: strong scaling.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Prints ONE JSON line on rank 0.  `--impl reference` times the fp64 CPU
oracle (oracle/, test infrastructure) on the host cores on a bounded sample of
the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

CFG = synth.CFG["cfg5"]
WORKLOAD = "cfg5: DP sparse MLP, 12x[768->3072 ReLU 3072->768] fp32, 95% uniform sparsity, " \
           "global batch 16384 tokens, MSE, SGD"


def fp32_peak_tflops(sm_mhz: float, sms: int = 148) -> float:
    """FP32 FMA peak = SMs x 128 FP32 lanes x 2 flop x clock."""
    return sms * 128 * 2 * sm_mhz * 1e6 / 1e12


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
def run_oracle_sample(target_s: float = 15.0):
    """The oracle as it stands, on the host cores, on a bounded sample of the
    cfg5 step: one block's six products (fwd W1 + ReLU, fwd W2, dW2, dZ, dW1,
    dX) on a token sample, repeated until ~target_s of CPU work.  Returns
    (GFLOP/s, cores, sample description, seconds)."""
    import oracle
    c = synth.mlp_case(blocks=1, d_model=CFG["d_model"], d_ff=CFG["d_ff"], T=2048,
                       density=CFG["density"], seed=CFG["seed"])
    w1, m1, w2, m2 = c["layers"][0]
    S1, S2 = oracle.csr_from_mask(w1, m1), oracle.csr_from_mask(w2, m2)
    nt = oracle.threads_available()
    T = 2048
    X = c["X0"][:, :T]
    tgt = c["target"][:, :T]
    flops_one = 6 * (S1.nnz + S2.nnz) * T
    t0 = time.perf_counter()
    reps = 0
    while True:
        Z = oracle.linear_fwd(S1, X, nt)
        H = np.maximum(Z, 0.0)
        Y = oracle.linear_fwd(S2, H, nt)
        dY = Y - tgt
        oracle.linear_bwd_weight(S2, H, dY, nt)
        dZ = oracle.linear_bwd_input(S2, dY, nt) * (H > 0)
        oracle.linear_bwd_weight(S1, X, dZ, nt)
        oracle.linear_bwd_input(S1, dZ, nt)
        reps += 1
        el = time.perf_counter() - t0
        if el >= target_s or reps >= 1000:
            break
    gflops = flops_one * reps / el / 1e9
    sample = (f"{reps} x one cfg5 block (6 products: fwd W1+ReLU, fwd W2, dW2, dX2*ReLU', dW1, dX1) "
              f"on {T} of 16384 tokens, fp64 oracle, {nt} OpenMP threads")
    return gflops, nt, sample, el


def reference_arm(args, rank: int, world: int):
    """--impl reference: the fp64 CPU oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return
    steps_t = []
    gfl = []
    nt = 1
    sample = ""
    per = max(3.0, 60.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        g, nt, sample, el = run_oracle_sample(per)
        if i >= args.warmup:
            steps_t.append(el)
            gfl.append(g)
    v = float(np.mean(gfl))
    line = {
        "impl": "reference", "metric": "sparse fwd+bwd effective GFLOP/s (2*nnz*B)", "value": v,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(steps_t)) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "global_batch": CFG["T"], "seq_len": None,
                   "parallelism": "none (host CPU)", "sample": sample},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": nt, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lr", type=float, default=1e-5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", type=int, default=None,
                    help="replay the whole step as one CUDA graph (default: 1 at N=1, 0 at N>1, where the "
                         "NCCL all_reduce would have to be captured too)")
    ap.add_argument("--sm-reserve", type=int, default=None,
                    help="N>1: SMs the backward's one-wave kernels leave to the all_reduce (default: 8 NCCL "
                         "channels; --comm p2p: the peer-memory kernel's CTAs)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "p2p", "nvls"],
                    help="N>1 dW all_reduce: NCCL, the library's peer-memory kernel, or its NVLS "
                         "multicast kernel (SURVEY F2)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config single-layer sweep (BASELINE configs 0-3) added at N=1")
    ap.add_argument("--tokens", type=int, default=CFG["T"], help="global batch (default 16384)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    assert args.warmup >= 3, "timing rules need >= 3 warm-up steps"
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_2302_04852_b200 import sparseprop as sp
    from paper_2302_04852_b200.dp import SparseMLP

    if args.sm_reserve is None:
        args.sm_reserve = sp.comm_ctas() if args.comm in ("p2p", "nvls") else 8
    if world > 1:
        # the dW all_reduce overlaps the backward: cap NCCL's CTAs (channels) and
        # leave that many SMs free in the one-wave kernels (SparseMLP sm_reserve)
        os.environ.setdefault("NCCL_MAX_NCHANNELS", str(args.sm_reserve))
        dist.init_process_group("nccl", device_id=dev)

    T = args.tokens
    lo, hi = synth.token_shard(T, world, rank)
    c = synth.mlp_case(blocks=CFG["blocks"], d_model=CFG["d_model"], d_ff=CFG["d_ff"], T=T,
                       density=CFG["density"], seed=CFG["seed"])
    model = SparseMLP(c["layers"], hi - lo, dev, sm_reserve=args.sm_reserve, comm=args.comm)
    # every rank must hold identical masks: allgather of a 64-bit hash of every
    # layer's (row_ptr, col_idx)
    if world > 1:
        import hashlib
        hh = hashlib.blake2b(digest_size=8)
        for W1, W2 in model.W:
            for Wh in (W1, W2):
                idx = Wh.indices()
                hh.update(idx["row_ptr"].cpu().numpy().tobytes())
                hh.update(idx["col_idx"].cpu().numpy().tobytes())
        hs = [None] * world
        dist.all_gather_object(hs, hh.hexdigest())
        assert len(set(hs)) == 1, "mask mismatch across ranks"

    X0_host = torch.from_numpy(np.ascontiguousarray(c["X0"][:, lo:hi])).pin_memory()
    T_host = torch.from_numpy(np.ascontiguousarray(c["target"][:, lo:hi])).pin_memory()
    model.set_batch(X0_host, T_host)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    # whole-step CUDA graphs (one per input-buffer parity, captured on first use,
    # outside every timed region) or eager launches
    use_graph = bool(args.graph if args.graph is not None else world == 1)
    graphs = {}

    def run_step():
        if not use_graph:
            return model.step(args.lr)
        key = (model.X[0].data_ptr(), model.target.data_ptr())
        g = graphs.get(key)
        if g is None:
            g = graphs[key] = model.capture(args.lr)
        g.replay()
        return model.loss

    # ---- device-timed region: inputs resident in HBM ---------------------
    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()
    n0 = sp.launch_count()
    model.step(args.lr)  # one eager (untimed) step: the library's launches per step
    torch.cuda.synchronize()
    launches_per_step = sp.launch_count() - n0
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    n0 = sp.launch_count()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        run_step()
    e1.record(stream)
    torch.cuda.synchronize()
    # graph replays re-launch the captured kernels without passing the host counter
    launches = launches_per_step * args.steps if use_graph else sp.launch_count() - n0
    ms = e0.elapsed_time(e1) / args.steps
    barrier()

    # ---- per-kernel breakdown (same stream, events around each launch) ----
    kt = {"fwd_spmm": [], "dx_spmm": [], "sddmm": [], "bwd_fused": []}
    ops = model.ops
    orig = {k: getattr(ops, k) for k in ("fwd", "dx", "dw", "bwd")}

    def wrap(name, key):
        f = orig[name]

        def g(*a, **k):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            r = f(*a, **k)
            e.record(stream)
            kt[key].append((s, e))
            return r
        return g
    ops.fwd, ops.dx, ops.dw = wrap("fwd", "fwd_spmm"), wrap("dx", "dx_spmm"), wrap("dw", "sddmm")
    ops.bwd = wrap("bwd", "bwd_fused")
    ksteps = max(3, min(args.steps, 10))
    for _ in range(ksteps):
        model.step(args.lr)
    torch.cuda.synchronize()
    ops.fwd, ops.dx, ops.dw, ops.bwd = orig["fwd"], orig["dx"], orig["dw"], orig["bwd"]
    clk = clocks.stop()
    ktime = {k: sum(s.elapsed_time(e) for s, e in v) / ksteps for k, v in kt.items() if v}  # ms per step

    # ---- end-to-end through the public API: host buffers in, loss out -----
    loss_host = torch.empty(1, pin_memory=True)
    # untimed warm-up of the e2e loop itself (same calls as the timed loop: the
    # staging buffers and the copy stream are created here, and the clocks are
    # up again after the idle gap of the clock-sampler teardown)
    def e2e_steps(n):
        model.prefetch_batch(X0_host, T_host)
        for k in range(n):
            model.use_prefetched()
            if k + 1 < n:
                model.prefetch_batch(X0_host, T_host)
            loss = run_step()
            model.release_staging()
            loss_host.copy_(loss, non_blocking=True)

    e2e_steps(args.warmup)
    torch.cuda.synchronize()
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    # every step's shard is copied from pinned host memory inside the timed
    # region; the copy of step k+1 runs on a side stream during step k (input
    # prefetch, double-buffered), and each step's loss is read back to the host
    e2e_steps(args.steps)
    e3.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e2.elapsed_time(e3) / args.steps
    h2d = (X0_host.numel() + T_host.numel()) * 4
    d2h = 4

    # ---- max over ranks ----------------------------------------------------
    t = torch.tensor([ms, ms_e2e], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ms_e2e = float(t[0]), float(t[1])
    flops_rank = model.step_flops()
    flops_all = torch.tensor([flops_rank], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(flops_all)
    flops_all = float(flops_all[0])
    value = flops_all / (ms * 1e-3) / 1e9
    value_e2e = flops_all / (ms_e2e * 1e-3) / 1e9

    if rank == 0:
        peaks = load_peaks()
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        fp32_peak = fp32_peak_tflops(sm_max)
        # dominant kernel class and its live roofline fraction
        dom = max(ktime, key=ktime.get)
        # fwd / dx / dw classes run one 2*nnz*B product per layer per step; the
        # fused backward runs two (dX and dW) per launch
        fl = sum(2 * (W1.nnz + W2.nnz) * model.T for W1, W2 in model.W) * (2 if dom == "bwd_fused" else 1)
        achieved = fl / (ktime[dom] * 1e-3) / 1e12
        # DRAM traffic per launch of this kernel from the committed ncu --set full capture
        traffic = None
        tf = os.path.join(ROOT, "profiles", "r2_kernel_traffic.json")
        if os.path.exists(tf):
            kt_ = json.load(open(tf)).get("kernels", {}).get(dom)
            if kt_:
                traffic = kt_["traffic_bytes_per_launch_mean"]
        step_roof_ms = model.step_flops() / (fp32_peak * 1e12) * 1e3
        line = {
            "metric": "sparse fwd+bwd effective GFLOP/s (2*nnz*B)", "value": value, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded PCG64, cfg5 shapes, random-init sparse weights)",
            "config": {"workload": WORKLOAD, "model": "sparse MLP 12x(768-3072-768) 95% sparse",
                       "global_batch": T, "seq_len": None, "parallelism": f"dp{world}",
                       "tokens_per_rank": hi - lo,
                       "dw_allreduce": (args.comm if world > 1 else "none (N=1)"),
                       "l2": "no flush: per-step working set (activations >= 300 MB per rank) > 126 MB L2",
                       "nnz_total": model.nnz_total},
            "roofline": {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": fp32_peak,
                         "unit": "TFLOP/s", "frac": achieved / fp32_peak, "traffic": traffic,
                         "traffic_unit": "bytes per launch (dram read + write, ncu --set full, profiles/)",
                         "peak_source": f"FP32 FMA: 148 SM x 128 lanes x 2 x {sm_max:.0f} MHz "
                                        f"(sm_max_mhz, {peaks['source']})",
                         "per_kernel_ms_per_step": ktime,
                         "step_frac_of_fp32_roofline": step_roof_ms / ms},
            "e2e": {"value": value_e2e, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d * world,
                    "d2h_bytes_per_step": d2h * world, "ms_per_step": ms_e2e,
                    "h2d": "pinned host -> device every step, next step's shard prefetched on a side stream"},
            "gpu_launches": int(launches),
            "cuda_graph": use_graph,
            "clocks": clk,
            "library": sp.version(),
        }
        if world == 1 and not args.no_configs:
            # driver-observed numbers for every single-layer BASELINE config
            # (cfg1, cfg2a/b, cfg3, the ten cfg4 instances) beside the cfg5 headline
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import config_sweep
            line["per_config"] = config_sweep.sweep(fp32_peak * 1e12, float(peaks.get("hbm_gbs", 6550.1)) * 1e9)
        if world == 1 and not args.no_cpu_baseline:
            g, nt, sample, _ = run_oracle_sample(15.0)
            line["cpu_baseline"] = {"value": g, "unit": "GFLOP/s", "cores": nt, "kind": "oracle",
                                    "sample": sample}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

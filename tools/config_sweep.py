"""Per-config measurements of the single-layer hot path (BASELINE.json configs
0-3: cfg1, cfg2a/2b, cfg3 and the ten cfg4 instances; plus, as context, the
paper's Fig. 3 layer 3072 x 768 at B = 902 over the same sparsity sweep) for bench.py's JSON line
(key "per_config") and for tools/ runs.

Each instance: forward + fused backward (sp_linear_fwd + sp_linear_bwd, conv:
sp_conv2d_fwd + sp_conv2d_bwd) through the C ABI on seeded synth inputs.
Timing: one CUDA graph per call, replayed after an L2 flush (a 256 MB write)
before every timed replay, CUDA events on the launching stream, median of
`reps`.  Two handle modes are timed:
  * managed (sp_weight_set_managed: vals change only through sp_weight_sgd, as
    in a training loop) -- the kernel path alone; this is the primary number;
  * api: an unmanaged handle, whose products first re-copy vals into the tiled
    index copies (one extra small kernel per product).
Effective FLOPs: 3 x 2*nnz*B (conv: exact valid taps).  Roofline
time: sum over the 3 products of max(FLOPs / FP32 peak, algorithmic bytes /
HBM).  `path` is sp_last_path() of each call (which kernels
ran).

Context column (not the library; SURVEY §8(d) "dense counterpart", the
paper's baseline P363-P366): the same layer dense in fp32 with TF32 off --
cuBLAS SGEMMs Y = W X, dX = W^T dY, dW = dY X^T (conv: cuDNN NCHW forward and
convolution_backward) on the masked weights, timed the same way;
`t_dense_us` and `speedup_vs_dense` = t_dense / t (the paper's Fig. 3 / 4
quantity on B200).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402

_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    _flush.fill_(1.0)


def graph_times(fns: dict, reps: int) -> dict:
    """Median device time (ms) of one graph replay of each fn, L2 flushed before each."""
    for _ in range(3):
        for f in fns.values():
            f()
    torch.cuda.synchronize()
    graphs = {}
    for k, f in fns.items():
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs[k] = g
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    out = {k: [] for k in fns}
    for _ in range(reps):
        for k, g in graphs.items():
            flush_l2()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            g.replay()
            e.record(st)
            e.synchronize()
            out[k].append(s.elapsed_time(e))
    return {k: float(np.median(v)) for k, v in out.items()}


class _NoTF32:
    """fp32 dense context runs: no TF32 in cuBLAS or cuDNN."""

    def __enter__(self):
        self.s = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False

    def __exit__(self, *a):
        torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = self.s


def dense_linear_us(Wm, X, dY, reps) -> float:
    R, C = Wm.shape
    B = X.shape[1]
    Yd, dXd = torch.empty(R, B, device="cuda"), torch.empty(C, B, device="cuda")
    dWd = torch.empty(R, C, device="cuda")
    with _NoTF32():
        t = graph_times({"fwd": lambda: torch.mm(Wm, X, out=Yd),
                         "bwd": lambda: (torch.mm(Wm.t(), dY, out=dXd), torch.mm(dY, X.t(), out=dWd))}, reps)
    return (t["fwd"] + t["bwd"]) * 1e3


def dense_conv_us(Wm, Xn, dYn, pad, reps) -> float:
    with _NoTF32():
        t = graph_times({"fwd": lambda: torch.nn.functional.conv2d(Xn, Wm, padding=pad),
                         "bwd": lambda: torch.ops.aten.convolution_backward(
                             dYn, Xn, Wm, None, [1, 1], [pad, pad], [1, 1], False, [0, 0], 1, [True, True, False])},
                        reps)
    return (t["fwd"] + t["bwd"]) * 1e3


def _paths(fns: dict) -> dict:
    p = {}
    for k, f in fns.items():
        f()
        p[k] = sp.last_path()
    torch.cuda.synchronize()
    return p


def linear(name, R, C, B, density, wvar, seed, kind="uniform", reps=7, peak=None, hbm=None):
    c = synth.linear_case(R, C, B, density, wvar, seed, kind)
    Wd, Md = torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda()
    X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
    Y, dX = torch.empty(R, B, device="cuda"), torch.empty(C, B, device="cuda")
    rec = {"config": name, "mask": kind, "sparsity": round(1 - density, 4), "R": R, "C": C, "B": B}
    for mode in ("managed", "api"):
        W = sp.sp_weight_create(Wd, Md)
        if mode == "managed":
            sp.sp_weight_set_managed(W, True)
        dW = torch.empty(max(W.nnz, 1), device="cuda")[:W.nnz]
        fns = {"fwd": lambda: sp.sp_linear_fwd(W, X, Y), "bwd": lambda: sp.sp_linear_bwd(W, X, dY, dX, dW)}
        t = graph_times(fns, reps)
        if mode == "managed":
            rec["nnz"] = W.nnz
            rec["path"] = _paths(fns)
            rec["t_fwd_us"] = round(t["fwd"] * 1e3, 2)
            rec["t_bwd_us"] = round(t["bwd"] * 1e3, 2)
            rec["t_us"] = round((t["fwd"] + t["bwd"]) * 1e3, 2)
        else:
            rec["t_api_us"] = round((t["fwd"] + t["bwd"]) * 1e3, 2)
        del W
    fl = 2 * rec["nnz"] * B
    nnz = rec["nnz"]
    byts = [8 * nnz + 4 * (R + 1) + 4 * B * (R + C), 8 * nnz + 4 * (C + 1) + 4 * B * (R + C),
            8 * nnz + 4 * B * (R + C) + 4 * nnz]
    roof = sum(max(fl / peak, b / hbm) for b in byts)
    tt = rec["t_us"] * 1e-6
    rec["gflops"] = round(3 * fl / tt / 1e9, 1)
    rec["roofline_us"] = round(roof * 1e6, 2)
    rec["pct_roofline"] = round(100 * roof / tt, 2)
    td = dense_linear_us(Wd * Md.to(torch.float32), X, dY, reps)
    rec["t_dense_us"] = round(td, 2)
    rec["speedup_vs_dense"] = round(td / rec["t_us"], 2)
    return rec


def conv(name, reps=7, peak=None, hbm=None, **cfg):
    c = synth.conv_case(**cfg)
    Wd, Md = torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda()
    X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
    Y = torch.empty(c["OC"], c["OH"], c["OW"], c["B"], device="cuda")
    dX = torch.empty_like(X)
    rec = {"config": name, "geom": f"{c['IC']}->{c['OC']} {c['H']}x{c['Wd']} k{c['KH']} pad{c['pad']}",
           "B": c["B"]}
    for mode in ("managed", "api"):
        W = sp.sp_weight_create(Wd, Md)
        if mode == "managed":
            sp.sp_weight_set_managed(W, True)
        g = sp.conv_geom(W, c["B"], c["H"], c["Wd"], c["pad"])
        dW = torch.empty(W.nnz, device="cuda")
        fns = {"fwd": lambda: sp.sp_conv2d_fwd(W, g, X, Y), "bwd": lambda: sp.sp_conv2d_bwd(W, g, X, dY, dX, dW)}
        t = graph_times(fns, reps)
        if mode == "managed":
            rec["nnz"] = W.nnz
            rec["path"] = _paths(fns)
            rec["t_fwd_us"] = round(t["fwd"] * 1e3, 2)
            rec["t_bwd_us"] = round(t["bwd"] * 1e3, 2)
            rec["t_us"] = round((t["fwd"] + t["bwd"]) * 1e3, 2)
        else:
            rec["t_api_us"] = round((t["fwd"] + t["bwd"]) * 1e3, 2)
        del W
    m = c["mask"].astype(bool)
    OH, OW, H, Wd_, pad = c["OH"], c["OW"], c["H"], c["Wd"], c["pad"]
    vp = np.array([sum(1 for p in range(OH) if 0 <= p + x - pad < H) for x in range(c["KH"])])
    vq = np.array([sum(1 for q in range(OW) if 0 <= q + y - pad < Wd_) for y in range(c["KW"])])
    taps = int((m.sum(axis=(0, 1)) * np.outer(vp, vq)).sum())
    fl = 2 * taps * c["B"]
    act = 4 * c["B"] * (c["IC"] * H * Wd_ + c["OC"] * OH * OW)
    nnz = rec["nnz"]
    byts = [8 * nnz + act, 8 * nnz + act, act + 4 * nnz]
    roof = sum(max(fl / peak, b / hbm) for b in byts)
    tt = rec["t_us"] * 1e-6
    rec["gflops_exact_taps"] = round(3 * fl / tt / 1e9, 1)
    rec["roofline_us"] = round(roof * 1e6, 2)
    rec["pct_roofline"] = round(100 * roof / tt, 2)
    # dense context: NCHW tensors, [OC][IC][KH][KW] masked weights
    Wn = (Wd * Md.to(torch.float32)).reshape(c["OC"], c["IC"], c["KH"], c["KW"]).contiguous()
    Xn = X.permute(3, 0, 1, 2).contiguous()
    dYn = dY.permute(3, 0, 1, 2).contiguous()
    td = dense_conv_us(Wn, Xn, dYn, pad, reps)
    rec["t_dense_us"] = round(td, 2)
    rec["speedup_vs_dense"] = round(td / rec["t_us"], 2)
    return rec


def linearity(recs, kind):
    """Least-squares fit of fwd+bwd time vs nnz over the cfg4 sweep (SPEC S578-S586 idea)."""
    pts = [(r["nnz"], r["t_us"]) for r in recs if r["config"] == "cfg4" and r.get("mask") == kind]
    if len(pts) < 3:
        return None
    x = np.array([p[0] for p in pts], dtype=np.float64)
    y = np.array([p[1] for p in pts], dtype=np.float64)
    A = np.vstack([x, np.ones_like(x)]).T
    (slope, icpt), *_ = np.linalg.lstsq(A, y, rcond=None)
    r2 = 1.0 - float(np.sum((y - A @ [slope, icpt]) ** 2)) / float(np.sum((y - y.mean()) ** 2))
    return {"mask": kind, "slope_us_per_Mnnz": round(slope * 1e6, 3), "intercept_us": round(icpt, 2),
            "r2": round(r2, 4), "points": len(pts)}


def sweep(peak_flops: float, hbm_bps: float, reps: int = 7, quick: bool = False) -> dict:
    kw = {"reps": reps, "peak": peak_flops, "hbm": hbm_bps}
    recs = [linear("cfg1", **synth.CFG["cfg1"], **kw)]
    for n in ("cfg2a", "cfg2b"):
        recs.append(linear(n, **synth.CFG[n], **kw))
    recs.append(conv("cfg3", **kw, **synth.CFG["cfg3"]))
    for kind in ("uniform", "zipf"):
        for s in synth.CFG4_SPARSITIES:
            cf = synth.cfg4(s, kind)
            recs.append(linear("cfg4", cf["R"], cf["C"], cf["B"], cf["density"], cf["wvar"], cf["seed"], kind, **kw))
            if quick:
                break
    if not quick:  # SURVEY §8(d) context: the paper's Fig. 3 layer (P366), B = 902, seeds 900 + s
        for s in synth.CFG4_SPARSITIES:
            recs.append(linear("ctx_paper_fig3", 3072, 768, 902, round(1.0 - s, 4), 1.0 / 768,
                               900 + int(round(s * 100)), "uniform", **kw))
    fits = [f for f in (linearity(recs, "uniform"), linearity(recs, "zipf")) if f]
    return {"timing": "CUDA-graph replay per call, L2 flushed (256 MB write) before each, median of "
                      f"{reps}; t_us = fwd + fused bwd, managed handle (no per-product vals refresh); "
                      "t_api_us = the same with an unmanaged handle; t_dense_us = the dense fp32 layer (cuBLAS / "
                      "cuDNN, TF32 off) fwd + bwd on the masked weights, context only",
            "instances": recs, "linearity": fits}


if __name__ == "__main__":
    import json
    pk = {"hbm_gbs": 6550.1, "sm_max_mhz": 1965.0}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        pk.update(json.load(open(p)))
    res = sweep(148 * 128 * 2 * pk["sm_max_mhz"] * 1e6, pk["hbm_gbs"] * 1e9, quick="--quick" in sys.argv)
    for r in res["instances"]:
        print(json.dumps(r))
    for f in res["linearity"]:
        print(json.dumps(f))

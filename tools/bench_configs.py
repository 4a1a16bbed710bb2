#!/usr/bin/env python
"""Per-config measurements of the single-layer hot path (BASELINE.json configs
0-3 and the paper's B=902 shape): fwd + dX + dW through the C ABI, CUDA-event
timed on the launching stream, L2 flushed before every timed repetition
(a 256 MB write), median of N.  Reports effective GFLOP/s (2*nnz*B per product;
conv: exact valid taps) and the roofline fraction
max(FLOPs / FP32 peak, algorithmic bytes / HBM) / time.
Writes JSON lines (one per config instance) to stdout or --out.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2302_04852_b200 import sparseprop as sp  # noqa: E402

PEAKS = {"hbm_gbs": 6550.1, "sm_max_mhz": 1965.0}
_p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(_p):
    PEAKS.update(json.load(open(_p)))
FP32 = 148 * 128 * 2 * PEAKS["sm_max_mhz"] * 1e6
HBM = PEAKS["hbm_gbs"] * 1e9

flush_buf = None


def flush_l2():
    global flush_buf
    if flush_buf is None:
        flush_buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    flush_buf.fill_(1.0)


def timed(fns, reps):
    """Per function: median over reps of (a) the CUDA-graph replay time of one
    call (kernel time, launch overhead removed) and (b) the event time around a
    direct API call (includes the host-side launch work), ms.  L2 is flushed
    before every timed repetition."""
    st = torch.cuda.current_stream()
    per = {k: [] for k in fns}
    api = {k: [] for k in fns}
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
    for _ in range(reps):
        for k, f in fns.items():
            for lst, call in ((per[k], graphs[k].replay), (api[k], f)):
                flush_l2()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(st)
                call()
                e.record(st)
                e.synchronize()
                lst.append(s.elapsed_time(e))
    return ({k: float(np.median(v)) for k, v in per.items()}, {k: float(np.median(v)) for k, v in api.items()})


def linear(name, R, C, B, density, wvar, seed, kind="uniform", reps=10, dense_ctx=True):
    c = synth.linear_case(R, C, B, density, wvar, seed, kind)
    W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
    X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
    Y, dX, dW = torch.empty(R, B, device="cuda"), torch.empty(C, B, device="cuda"), torch.empty(max(W.nnz, 1), device="cuda")
    t, ta = timed({"fwd": lambda: sp.sp_linear_fwd(W, X, Y), "dx": lambda: sp.sp_linear_bwd_input(W, dY, dX),
                   "dw": lambda: sp.sp_linear_bwd_weight(W, X, dY, dW[:W.nnz]),
                   "bwd_fused": lambda: sp.sp_linear_bwd(W, X, dY, dX, dW[:W.nnz])}, reps)
    tf = t.pop("bwd_fused")
    taf = ta.pop("bwd_fused")
    fl = 2 * W.nnz * B
    byts = {"fwd": 8 * W.nnz + 4 * (R + 1) + 4 * B * (R + C), "dx": 8 * W.nnz + 4 * (C + 1) + 4 * B * (R + C),
            "dw": 8 * W.nnz + 4 * B * (R + C) + 4 * W.nnz}
    rec = {"config": name, "mask": kind, "sparsity": round(1 - density, 4), "R": R, "C": C, "B": B, "nnz": W.nnz,
           "seed": seed, "l2": "flushed before each timed launch", "timing": "CUDA-graph replay of one call (t_*), direct API call (t_api_*)"}
    tot_t = sum(t.values())
    roof = sum(max(fl / FP32, byts[k] / HBM) for k in t)
    rec.update({f"t_{k}_us": round(v * 1e3, 2) for k, v in t.items()})
    rec["t_fwd_bwd_us"] = round(tot_t * 1e3, 2)
    rec["t_fwd_bwd_fused_us"] = round((t["fwd"] + tf) * 1e3, 2)  # fwd + fused dX/dW (sp_linear_bwd)
    rec["t_api_fwd_bwd_us"] = round(sum(ta.values()) * 1e3, 2)  # direct API calls incl. host launch work
    rec["eff_gflops"] = round(3 * fl / (tot_t * 1e-3) / 1e9, 1)
    rec["eff_gflops_fused"] = round(3 * fl / ((t["fwd"] + tf) * 1e-3) / 1e9, 1)
    rec["roofline_us"] = round(roof * 1e6, 2)
    rec["pct_roofline"] = round(100 * roof / (tot_t * 1e-3), 2)
    rec["pct_roofline_fused"] = round(100 * roof / ((t["fwd"] + tf) * 1e-3), 2)  # fwd + sp_linear_bwd
    rec["pct_fp32_peak"] = round(100 * 3 * fl / (tot_t * 1e-3) / FP32, 2)
    if dense_ctx:  # the paper's "dense counterpart" (P363): cuBLAS fp32, TF32 off, masked W
        torch.backends.cuda.matmul.allow_tf32 = False
        Wd = torch.from_numpy(c["W"] * c["mask"]).cuda()
        td, _ = timed({"fwd": lambda: Wd @ X, "dx": lambda: Wd.t() @ dY, "dw": lambda: dY @ X.t()}, reps)
        rec["dense_cublas_fp32_us"] = round(sum(td.values()) * 1e3, 2)
    return rec


def conv(name, reps=10, **cfg):
    c = synth.conv_case(**cfg)
    W = sp.sp_weight_create(torch.from_numpy(c["W"]).cuda(), torch.from_numpy(c["mask"]).cuda())
    g = sp.conv_geom(W, c["B"], c["H"], c["Wd"], c["pad"])
    X, dY = torch.from_numpy(c["X"]).cuda(), torch.from_numpy(c["dY"]).cuda()
    Y = torch.empty(c["OC"], c["OH"], c["OW"], c["B"], device="cuda")
    dX = torch.empty_like(X)
    dW = torch.empty(W.nnz, device="cuda")
    t, ta = timed({"fwd": lambda: sp.sp_conv2d_fwd(W, g, X, Y), "dx": lambda: sp.sp_conv2d_bwd_input(W, g, dY, dX),
                   "dw": lambda: sp.sp_conv2d_bwd_weight(W, g, X, dY, dW),
                   "bwd_fused": lambda: sp.sp_conv2d_bwd(W, g, X, dY, dX, dW)}, reps)
    tf = t.pop("bwd_fused")
    ta.pop("bwd_fused")
    # exact useful FMAs: per tap (x, y), valid output rows x cols (C20)
    m = c["mask"].astype(bool)
    OH, OW, H, Wd, pad = c["OH"], c["OW"], c["H"], c["Wd"], c["pad"]
    vp = np.array([sum(1 for p in range(OH) if 0 <= p + x - pad < H) for x in range(c["KH"])])
    vq = np.array([sum(1 for q in range(OW) if 0 <= q + y - pad < Wd) for y in range(c["KW"])])
    taps = (m.sum(axis=(0, 1)) * np.outer(vp, vq)).sum()
    fl = 2 * int(taps) * c["B"]
    fl_nominal = 2 * W.nnz * c["B"] * OH * OW
    act = 4 * c["B"] * (c["IC"] * H * Wd + c["OC"] * OH * OW)
    byts = {"fwd": 8 * W.nnz + act, "dx": 8 * W.nnz + act, "dw": act + 4 * W.nnz}
    tot_t = sum(t.values())
    roof = sum(max(fl / FP32, byts[k] / HBM) for k in t)
    rec = {"config": name, "nnz": W.nnz, "B": c["B"], "geom": f"{c['IC']}->{c['OC']} {H}x{Wd} k{c['KH']} pad{pad}",
           "l2": "flushed before each timed launch", "timing": "CUDA-graph replay of one call (t_*), direct API call (t_api_*)"}
    rec.update({f"t_{k}_us": round(v * 1e3, 2) for k, v in t.items()})
    rec["t_fwd_bwd_us"] = round(tot_t * 1e3, 2)
    rec["t_fwd_bwd_fused_us"] = round((t["fwd"] + tf) * 1e3, 2)  # fwd + sp_conv2d_bwd
    rec["t_api_fwd_bwd_us"] = round(sum(ta.values()) * 1e3, 2)
    rec["eff_gflops_exact_fused"] = round(3 * fl / ((t["fwd"] + tf) * 1e-3) / 1e9, 1)
    rec["pct_roofline_fused"] = round(100 * sum(max(fl / FP32, byts[k] / HBM) for k in byts) / ((t["fwd"] + tf) * 1e-3), 2)
    rec["eff_gflops_exact"] = round(3 * fl / (tot_t * 1e-3) / 1e9, 1)
    rec["eff_gflops_nominal"] = round(3 * fl_nominal / (tot_t * 1e-3) / 1e9, 1)
    rec["roofline_us"] = round(roof * 1e6, 2)
    rec["pct_roofline"] = round(100 * roof / (tot_t * 1e-3), 2)
    # dense cuDNN fp32 context (NCHW)
    torch.backends.cudnn.allow_tf32 = False
    Xn = X.permute(3, 0, 1, 2).contiguous()
    Wm = torch.from_numpy(c["W"] * c["mask"]).cuda()
    td, _ = timed({"fwd": lambda: torch.nn.functional.conv2d(Xn, Wm, padding=pad)}, reps)
    rec["dense_cudnn_fp32_fwd_us"] = round(td["fwd"] * 1e3, 2)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    recs = []
    recs.append(linear("cfg1", **synth.CFG["cfg1"], reps=a.reps))
    for n in ("cfg2a", "cfg2b"):
        recs.append(linear(n, **synth.CFG[n], reps=a.reps))
    recs.append(conv("cfg3", reps=a.reps, **synth.CFG["cfg3"]))
    for kind in ("uniform", "zipf"):
        for s in synth.CFG4_SPARSITIES:
            cf = synth.cfg4(s, kind)
            recs.append(linear("cfg4", cf["R"], cf["C"], cf["B"], cf["density"], cf["wvar"], cf["seed"], kind,
                               reps=a.reps))
            if a.quick:
                break
    recs.append(linear("paper_B902", 3072, 768, 902, 0.1, 1.0 / 768, 990, reps=a.reps))
    # runtime linear in nnz (SPEC S578-S586 idea): least-squares fit over the cfg4 sweep
    for kind in ("uniform", "zipf"):
        pts = [(r["nnz"], r["t_fwd_bwd_us"]) for r in recs if r["config"] == "cfg4" and r.get("mask") == kind]
        if len(pts) >= 3:
            x = np.array([p[0] for p in pts], dtype=np.float64)
            y = np.array([p[1] for p in pts], dtype=np.float64)
            A = np.vstack([x, np.ones_like(x)]).T
            (slope, icpt), *_ = np.linalg.lstsq(A, y, rcond=None)
            r2 = 1.0 - float(np.sum((y - A @ [slope, icpt]) ** 2)) / float(np.sum((y - y.mean()) ** 2))
            recs.append({"config": "cfg4_linearity", "mask": kind, "slope_us_per_Mnnz": round(slope * 1e6, 3),
                         "intercept_us": round(icpt, 2), "r2": round(r2, 4), "points": len(pts)})
    out = open(a.out, "w") if a.out else sys.stdout
    for r in recs:
        out.write(json.dumps(r) + "\n")
        out.flush()


if __name__ == "__main__":
    main()

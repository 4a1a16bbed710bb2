"""Graph-replayed, L2-flushed timings (config_sweep's method) of chosen
single-layer configs, for A/B runs:  python tools/cfg_time.py cfg2a cfg4:uniform:0.99 ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import config_sweep as cs  # noqa: E402
import synth  # noqa: E402

PEAK, HBM = 148 * 128 * 2 * 1965e6, 6550.1e9
for name in sys.argv[1:]:
    if name.startswith("cfg4:"):  # cfg4:kind:sparsity[:B]
        _, kind, sp_, *rest = name.split(":")
        cf = synth.cfg4(float(sp_), kind)
        B = int(rest[0]) if rest else cf["B"]
        r = cs.linear("cfg4" + (f"@B{B}" if rest else ""), cf["R"], cf["C"], B, cf["density"], cf["wvar"], cf["seed"],
                      kind, reps=9, peak=PEAK, hbm=HBM)
    elif name.startswith("ctx:"):  # ctx:sparsity[:B] -- the paper's Fig. 3 layer, B = 902 by default
        _, sp_, *rest = name.split(":")
        s100 = int(round(float(sp_) * 100))
        B = int(rest[0]) if rest else 902
        r = cs.linear(f"ctx@B{B}", 3072, 768, B, round(1 - float(sp_), 4), 1.0 / 768, 900 + s100, "uniform",
                      reps=9, peak=PEAK, hbm=HBM)
    elif name in ("cfg5w1", "cfg5w2"):  # the bench's layer shapes at the full 16384 tokens
        R, C = (3072, 768) if name == "cfg5w1" else (768, 3072)
        r = cs.linear(name, R, C, 16384, 0.05, 1.0 / C, 5, reps=5, peak=PEAK, hbm=HBM)
    elif name == "cfg3":
        r = cs.conv("cfg3", reps=9, peak=PEAK, hbm=HBM, **synth.CFG["cfg3"])
    elif "@" in name:  # cfg2a@B: a cfg2 shape at another batch
        base, B = name.split("@")
        cf = dict(synth.CFG[base])
        cf["B"] = int(B)
        r = cs.linear(name, **cf, reps=9, peak=PEAK, hbm=HBM)
    else:
        r = cs.linear(name, **synth.CFG[name], reps=9, peak=PEAK, hbm=HBM)
    print(json.dumps({k: r[k] for k in ("config", "t_fwd_us", "t_bwd_us", "t_us", "pct_roofline", "path")
                      if k in r} | {"mask": r.get("mask"), "sparsity": r.get("sparsity")}), flush=True)

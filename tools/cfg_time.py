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
    if name.startswith("cfg4:"):
        _, kind, sp_ = name.split(":")
        cf = synth.cfg4(float(sp_), kind)
        r = cs.linear("cfg4", cf["R"], cf["C"], cf["B"], cf["density"], cf["wvar"], cf["seed"], kind, reps=9,
                      peak=PEAK, hbm=HBM)
    elif name == "cfg3":
        r = cs.conv("cfg3", reps=9, peak=PEAK, hbm=HBM, **synth.CFG["cfg3"])
    else:
        r = cs.linear(name, **synth.CFG[name], reps=9, peak=PEAK, hbm=HBM)
    print(json.dumps({k: r[k] for k in ("config", "t_fwd_us", "t_bwd_us", "t_us", "pct_roofline", "path")
                      if k in r} | {"mask": r.get("mask"), "sparsity": r.get("sparsity")}), flush=True)

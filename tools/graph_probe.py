"""Is the per-rank cfg5 step host-bound at small token shares?  Times (CUDA
events, 10 steps after warm-up) the step run directly and replayed from a CUDA
graph captured once (forward + backward + managed SGD), for T tokens."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2302_04852_b200.dp import SparseMLP  # noqa: E402

CFG = synth.CFG["cfg5"]
for T in (2048, 4096, 16384):
    c = synth.mlp_case(blocks=CFG["blocks"], d_model=CFG["d_model"], d_ff=CFG["d_ff"], T=T,
                       density=CFG["density"], seed=CFG["seed"])
    m = SparseMLP(c["layers"], T, "cuda")
    m.set_batch(torch.from_numpy(c["X0"]), torch.from_numpy(c["target"]), non_blocking=False)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(5):
            m.step(1e-5)
    torch.cuda.synchronize()

    def timed(fn, n=10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            for _ in range(n):
                fn()
            b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    direct = timed(lambda: m.step(1e-5))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        m.step(1e-5)
    torch.cuda.synchronize()
    replay = timed(g.replay)
    print(f"T={T:6d}: direct {direct:7.3f} ms  graph replay {replay:7.3f} ms  ({(direct / replay - 1) * 100:+.1f} %)",
          flush=True)
    del m, g
    torch.cuda.empty_cache()

"""Where does the e2e step lose time against the device-resident step?
Times (CUDA events, 10 steps after 5 warm-up) the cfg5 step: (a) inputs
resident, (b) e2e as bench.py does it (prefetched H2D + loss D2H), (c) e2e
without the loss read-back, (d) H2D copies alone on the side stream."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2302_04852_b200.dp import SparseMLP  # noqa: E402

CFG = synth.CFG["cfg5"]
c = synth.mlp_case(blocks=CFG["blocks"], d_model=CFG["d_model"], d_ff=CFG["d_ff"], T=CFG["T"],
                   density=CFG["density"], seed=CFG["seed"])
m = SparseMLP(c["layers"], CFG["T"], "cuda")
X0 = torch.from_numpy(np.ascontiguousarray(c["X0"])).pin_memory()
Tt = torch.from_numpy(np.ascontiguousarray(c["target"])).pin_memory()
m.set_batch(X0, Tt)
st = torch.cuda.current_stream()
loss_host = torch.empty(1, pin_memory=True)


def timed(fn, steps=10):
    for _ in range(5):
        fn(0, steps)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for k in range(steps):
        fn(k, steps)
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def resident(k, n):
    m.step(1e-5)


def e2e(k, n, readback=True):
    if k == 0:
        m.prefetch_batch(X0, Tt)
    m.use_prefetched()
    if k + 1 < n:
        m.prefetch_batch(X0, Tt)
    loss = m.step(1e-5)
    m.release_staging()
    if readback:
        loss_host.copy_(loss, non_blocking=True)


cs = torch.cuda.Stream()
buf = (torch.empty_like(m.X[0]), torch.empty_like(m.target))


def h2d(k, n):
    with torch.cuda.stream(cs):
        buf[0].copy_(X0, non_blocking=True)
        buf[1].copy_(Tt, non_blocking=True)
    st.wait_stream(cs)


print(f"resident step      {timed(resident):8.3f} ms")
print(f"e2e (bench)        {timed(e2e):8.3f} ms")
print(f"e2e, no read-back  {timed(lambda k, n: e2e(k, n, False)):8.3f} ms")
print(f"H2D alone (100 MB) {timed(h2d):8.3f} ms")
print(f"resident step      {timed(resident):8.3f} ms")

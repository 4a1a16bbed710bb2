"""From-scratch sparse training with gradual magnitude pruning (
the paper's §4.2.2 schedule, P559-P560): "train the model dense for ten epochs
before pruning the lowest 5% of the weights (either uniformly or globally)
and then prune gradually every 10 epochs until epoch 80, at which point we
fine-tune for a further 20 epochs".

Synthetic stand-in for the paper's datasets (none is available): a student
MLP of SparseLinear modules (2 x [768 -> 3072, ReLU, 3072 -> 768], the cfg5
block) regresses the outputs of a fixed random dense teacher of the same
shape on N(0,1) inputs, MSE loss, SGD with momentum.  An "epoch" is
--steps-per-epoch optimizer steps of --batch tokens.  At every pruning epoch
the modules are pruned by magnitude to gmp_target_at(epoch) (uniform or
global) and rebuilt through sp_weight_create; the record of each update holds
the rebuild time (the handle-creation cost the paper's "masks change only a
few times" argument, P428, amortises), the achieved sparsities, and the §4.2
dispatcher's decision and probe timings (P427-P429) of every module.

  python tools/gmp_train.py [--final 0.95] [--scope uniform|global] [--out profiles/r2_gmp_train.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_04852_b200.nn import SparseLinear  # noqa: E402
from paper_2302_04852_b200.prune import gmp_target_at, prune_modules  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--final", type=float, default=0.95)
    ap.add_argument("--scope", default="uniform", choices=["uniform", "global"])
    ap.add_argument("--epochs", type=int, default=100)
    ap.add_argument("--steps-per-epoch", type=int, default=20)
    ap.add_argument("--batch", type=int, default=2048)
    ap.add_argument("--blocks", type=int, default=2)
    ap.add_argument("--lr", type=float, default=2e-3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(2302)
    dm, dff = 768, 3072
    # fixed random dense teacher
    teacher = []
    for _ in range(a.blocks):
        teacher.append((torch.randn(dff, dm, generator=g, device=dev) / dm ** 0.5,
                        torch.randn(dm, dff, generator=g, device=dev) * (2.0 / dff) ** 0.5))

    def teach(x):  # x [N, dm]
        for w1, w2 in teacher:
            x = torch.relu(x @ w1.t()) @ w2.t()
        return x

    # dense-initialised student: SparseLinear with an all-ones mask (sparsity 0: the
    # dispatcher runs it dense until pruning makes it >= 80 % sparse)
    mods = []
    for _ in range(a.blocks):
        w1 = torch.randn(dff, dm, generator=g, device=dev) / dm ** 0.5
        w2 = torch.randn(dm, dff, generator=g, device=dev) * (2.0 / dff) ** 0.5
        mods.append(SparseLinear(w1, torch.ones_like(w1, dtype=torch.uint8)))
        mods.append(SparseLinear(w2, torch.ones_like(w2, dtype=torch.uint8)))
    params = [m.vals for m in mods]
    opt = torch.optim.SGD(params, lr=a.lr, momentum=0.9)

    def student(x):
        for i in range(0, len(mods), 2):
            x = mods[i + 1](torch.relu(mods[i](x)))
        return x

    out = open(a.out, "w") if a.out else None

    def emit(rec):
        line = json.dumps(rec)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()

    emit({"event": "start", "model": f"{a.blocks} x [768->3072 ReLU 3072->768] SparseLinear student vs dense teacher",
          "schedule": "GMP (P559-P560): dense 10 epochs, prune 5% at epoch 10, every 10 epochs to epoch 80 "
                      "(cubic interpolation, SPEC S432), fine-tune 20", "final": a.final, "scope": a.scope,
          "epochs": a.epochs, "steps_per_epoch": a.steps_per_epoch, "batch": a.batch})
    cur = 0.0
    t_train = time.perf_counter()
    for ep in range(a.epochs):
        target = gmp_target_at(ep, a.final)
        if target > cur + 1e-12:
            loss = None  # release the last step's autograd graph before vals change size
            rep = prune_modules(mods, target, scope=a.scope, optimizer=opt)
            cur = target
            x0 = torch.randn(a.batch, dm, generator=g, device=dev)
            student(x0)  # the first call after a mask change runs the dispatcher probe (P428)
            torch.cuda.synchronize()
            emit({"event": "prune", "epoch": ep, "target": round(target, 4),
                  "achieved": [round(s, 4) for s in rep["sparsity"]], "rebuild_ms": round(rep["rebuild_s"] * 1e3, 2),
                  "rebuild_ms_per_module": round(rep["rebuild_s"] * 1e3 / len(mods), 2),
                  "impl": [m.impl for m in mods],
                  "probe_ms": [{k: round(v, 3) for k, v in (m.probe_ms or {}).items()} for m in mods]})
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        losses = []
        for _ in range(a.steps_per_epoch):
            x = torch.randn(a.batch, dm, generator=g, device=dev)
            y = teach(x)
            loss = torch.nn.functional.mse_loss(student(x), y)
            opt.zero_grad(set_to_none=True)
            loss.backward()
            opt.step()
            losses.append(loss.detach())
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / a.steps_per_epoch
        if ep % 5 == 0 or ep == a.epochs - 1 or target != gmp_target_at(ep + 1, a.final):
            emit({"event": "epoch", "epoch": ep, "sparsity": round(cur, 4),
                  "loss": round(float(torch.stack(losses).mean()), 6), "ms_per_step": round(ms, 3),
                  "impl": sorted(set(m.impl for m in mods))})
    emit({"event": "end", "train_s": round(time.perf_counter() - t_train, 1),
          "final_sparsity": [round(1 - m.W.nnz / float(m.W.R * m.W.C), 4) for m in mods]})


if __name__ == "__main__":
    main()

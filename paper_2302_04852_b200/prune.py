"""Magnitude pruning and the gradual-magnitude-pruning (GMP) schedule of the
paper's from-scratch experiments (§4.2.2, P559-P560): "train the model dense
for ten epochs before pruning the lowest 5% of the weights (either uniformly or
globally) and then prune gradually every 10 epochs until epoch 80, at which
point we fine-tune for a further 20 epochs".

These run a few times per training run (masks "change only a few times",
P428), off the hot path: mask selection is a sort of |w| (torch), after which
the affected modules rebuild their sparse structure with sp_weight_create
(`SparseLinear.set_mask`), whose cost `prune_modules` reports.

Readings: the paper gives only the 5 % start and the 10-epoch
cadence; the interpolation between 5 % and the target is the cubic schedule of
the GMP method it cites (SPEC S429-S437), held constant between pruning
epochs; ties in |w| keep the smaller flat index (deterministic).
"""
from __future__ import annotations

import math
import time

import torch


def gmp_target_at(epoch: int, final: float, start: int = 10, end: int = 80, every: int = 10,
                  initial: float = 0.05) -> float:
    """Sparsity in force at `epoch`: 0 before `start`; at the pruning epochs
    start, start+every, ..., end the cubic s_i + (s_f - s_i)(1 - (1 - t)^3),
    t = (e - start)/(end - start); constant in between and after `end`."""
    if epoch < start:
        return 0.0
    e = min(epoch - (epoch - start) % every, end)
    t = (e - start) / float(end - start)
    return initial + (final - initial) * (1.0 - (1.0 - t) ** 3)


def _n_keep(sparsity: float, n: int) -> int:
    """ceil((1 - s) n), robust to the binary representation of s (0.95 etc.)."""
    return min(n, math.ceil((1.0 - sparsity) * n - 1e-9))


def _keep_top(scores: torch.Tensor, n_keep: int) -> torch.Tensor:
    """Boolean mask keeping the n_keep largest scores (ties: smaller index first)."""
    flat = scores.flatten()
    order = torch.sort(-flat, stable=True).indices  # descending score, ascending index on ties
    keep = torch.zeros_like(flat, dtype=torch.bool)
    keep[order[:n_keep]] = True
    return keep.view(scores.shape)


def magnitude_mask(weight: torch.Tensor, sparsity: float, current: torch.Tensor | None = None) -> torch.Tensor:
    """Uniform (per-layer) magnitude pruning: keep ceil((1 - s) * n) largest |w|
    among the currently kept entries (all, if `current` is None)."""
    if not 0.0 <= sparsity < 1.0:
        raise ValueError("sparsity must be in [0, 1)")
    scores = weight.detach().abs().float()
    if current is not None:
        scores = torch.where(current.bool(), scores, torch.full_like(scores, -1.0))
    return _keep_top(scores, _n_keep(sparsity, weight.numel()))


def global_magnitude_masks(weights: list[torch.Tensor], sparsity: float,
                           currents: list[torch.Tensor] | None = None) -> list[torch.Tensor]:
    """Global magnitude pruning: one ranking of |w| over all layers jointly."""
    if not weights:
        raise ValueError("empty layer list")
    scores = []
    for i, w in enumerate(weights):
        s = w.detach().abs().float().flatten()
        if currents is not None:
            s = torch.where(currents[i].bool().flatten(), s, torch.full_like(s, -1.0))
        scores.append(s)
    allsc = torch.cat(scores)
    keep = _keep_top(allsc, _n_keep(sparsity, allsc.numel()))
    out, off = [], 0
    for w in weights:
        out.append(keep[off:off + w.numel()].view(w.shape))
        off += w.numel()
    return out


def prune_modules(modules, sparsity: float, scope: str = "uniform", optimizer=None) -> dict:
    """Prune SparseLinear / SparseConv2d modules to `sparsity` by magnitude of
    their current kept weights and rebuild their sparse structure.  Each
    module keeps its `vals` Parameter object (re-pointed at the new handle),
    so `optimizer` keeps stepping it; its per-parameter state, whose size
    was the old nnz, is dropped.  Autograd graphs recorded before the update
    must have been released (a live loss tensor from the last step still holds
    the old-size gradient accumulator of `vals`).  Returns the achieved
    sparsities and the time spent rebuilding (the sp_weight_create cost this
    mask update pays)."""
    dense, cur = [], []
    for m in modules:
        shape = m.W.filter_shape or (m.W.R, m.W.C)
        dense.append(m.W.to_dense(m.vals.detach()).view(shape))
        cur.append((m.W.to_dense(torch.ones_like(m.vals.detach())) != 0).view(shape))  # the current mask
    if scope == "uniform":
        masks = [magnitude_mask(d, sparsity, c) for d, c in zip(dense, cur)]
    elif scope == "global":
        masks = global_magnitude_masks(dense, sparsity, cur)
    else:
        raise ValueError(scope)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for m, d, k in zip(modules, dense, masks):
        m.set_mask(d * k, k.to(torch.uint8))
    torch.cuda.synchronize()
    rebuild_s = time.perf_counter() - t0
    if optimizer is not None:
        for m in modules:
            optimizer.state.pop(m.vals, None)
    achieved = [1.0 - m.W.nnz / float(m.W.R * m.W.C) for m in modules]
    return {"sparsity": achieved, "rebuild_s": rebuild_s}

"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no products, no gradients, no
index structure): it only draws masks, weights and activations with numpy's
PCG64 generator, in the fixed order mask -> values -> X -> dY (-> targets)
(SURVEY.md §8(d) "Synthetic inputs").  Both sides of every parity check
receive the same arrays from here; neither side imports the other.

Readings (listed in DESIGN.md §3):
  * N(0, v): the second parameter is the VARIANCE.
  * Masks are iid Bernoulli(density) unless a Zipf row profile is asked for
    (C14, the "rank-profile" reading of BASELINE.json configs[3]).
  * Off-mask dense values are drawn too (nonzero junk): structure comes from
    the mask only (C10), so a kernel that reads them is caught.

Layouts: linear activations are [features x B] row-major
(batch contiguous, the paper's X^T, PAPER.md P183 §3.2); conv activations are
CHWN [C][H][W][B] (the paper's batch-last layout, P293 §3.3).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "rng", "bernoulli_mask", "zipf_row_counts", "zipf_mask", "normal",
    "linear_case", "conv_case", "mlp_case", "CFG",
]


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def bernoulli_mask(g: np.random.Generator, R: int, C: int, density: float) -> np.ndarray:
    """iid Bernoulli(density) mask, uint8 R x C (1 = kept)."""
    return (g.random((R, C)) < density).astype(np.uint8)


def normal(g: np.random.Generator, shape, var: float) -> np.ndarray:
    """fp32 draws of N(0, var) (var is the variance, C13)."""
    return (g.standard_normal(shape) * np.sqrt(var)).astype(np.float32)


def zipf_row_counts(g: np.random.Generator, R: int, C: int, density: float,
                    s: float = 1.2) -> np.ndarray:
    """Per-row nnz following a Zipf(s) rank profile rescaled to the target density.

    SURVEY §8(c) C14 reading: a seeded permutation pi of 1..R gives row weight
    w_i = pi(i)^-s; n_i = min(C, floor(a * w_i)) with a found by bisection so that
    sum n_i <= round(density*R*C); the remainder goes +1 to unclipped rows by
    largest fractional part (ties -> lower row).  Exact total, 0 <= n_i <= C.
    """
    target = int(round(density * R * C))
    pi = g.permutation(R) + 1
    w = pi.astype(np.float64) ** (-s)

    def total(a):
        return int(np.minimum(C, np.floor(a * w)).sum())

    lo, hi = 0.0, 1.0
    while total(hi) < target and hi < 1e30:
        hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if total(mid) <= target:
            lo = mid
        else:
            hi = mid
    raw = lo * w
    n = np.minimum(C, np.floor(raw)).astype(np.int64)
    rem = target - int(n.sum())
    if rem > 0:
        frac = np.where(n < C, raw - np.floor(raw), -1.0)
        order = np.lexsort((np.arange(R), -frac))  # largest frac first, ties -> lower row
        cand = [i for i in order if n[i] < C][:rem]
        n[np.array(cand, dtype=np.int64)] += 1
    return n


def zipf_mask(g: np.random.Generator, R: int, C: int, density: float, s: float = 1.2) -> np.ndarray:
    n = zipf_row_counts(g, R, C, density, s)
    m = np.zeros((R, C), dtype=np.uint8)
    for r in range(R):
        if n[r]:
            m[r, g.choice(C, size=int(n[r]), replace=False)] = 1
    return m


# ---------------------------------------------------------------------------
# BASELINE.json configs (SURVEY §8(d) table "Synthetic inputs")
# ---------------------------------------------------------------------------
CFG = {
    "cfg1": dict(R=256, C=256, B=32, density=0.10, wvar=1.0 / 256, seed=1),
    "cfg2a": dict(R=3072, C=768, B=512, density=0.05, wvar=1.0 / 768, seed=21),
    "cfg2b": dict(R=768, C=3072, B=512, density=0.05, wvar=1.0 / 768, seed=22),
    "cfg3": dict(OC=256, IC=256, H=14, W=14, KH=3, KW=3, pad=1, B=64, density=0.10,
                 wvar=2.0 / 2304, seed=3),
    "cfg5": dict(blocks=12, d_model=768, d_ff=3072, T=16384, density=0.05, seed=5),
}
CFG4_SPARSITIES = (0.80, 0.90, 0.95, 0.98, 0.99)


def cfg4(sparsity: float, kind: str = "uniform") -> dict:
    s100 = int(round(sparsity * 100))
    seed = (400 if kind == "uniform" else 500) + s100
    return dict(R=4096, C=4096, B=256, density=1.0 - sparsity, wvar=1.0 / 4096, seed=seed,
                kind=kind)


def linear_case(R: int, C: int, B: int, density: float, wvar: float, seed: int,
                kind: str = "uniform") -> dict:
    """One sparse linear layer: W dense R x C fp32 (+junk off-mask), mask u8,
    X [C x B], dY [R x B] ~ N(0,1).  Draw order: mask, W, X, dY."""
    g = rng(seed)
    if kind == "uniform":
        mask = bernoulli_mask(g, R, C, density)
    elif kind == "zipf":
        mask = zipf_mask(g, R, C, density)
    else:
        raise ValueError(kind)
    W = normal(g, (R, C), wvar)
    X = normal(g, (C, B), 1.0)
    dY = normal(g, (R, B), 1.0)
    return dict(W=W, mask=mask, X=X, dY=dY, R=R, C=C, B=B)


def conv_case(OC: int, IC: int, H: int, W: int, KH: int, KW: int, pad: int, B: int,
              density: float, wvar: float, seed: int) -> dict:
    """Sparse conv layer (stride 1): weight [OC][IC][KH][KW] (+ mask), X CHWN
    [IC][H][W][B], dY CHWN [OC][OH][OW][B], OH = H + 2 pad - KH + 1."""
    g = rng(seed)
    OH, OW = H + 2 * pad - KH + 1, W + 2 * pad - KW + 1
    mask = (g.random((OC, IC, KH, KW)) < density).astype(np.uint8)
    Wt = normal(g, (OC, IC, KH, KW), wvar)
    X = normal(g, (IC, H, W, B), 1.0)
    dY = normal(g, (OC, OH, OW, B), 1.0)
    return dict(W=Wt, mask=mask, X=X, dY=dY, OC=OC, IC=IC, H=H, Wd=W, KH=KH, KW=KW,
                pad=pad, B=B, OH=OH, OW=OW)


def mlp_case(blocks: int, d_model: int, d_ff: int, T: int, density: float, seed: int,
             with_data: bool = True) -> dict:
    """cfg5: `blocks` x [W1 d_ff x d_model, ReLU, W2 d_model x d_ff].

    Init (variance preserving on the kept weights):
    W1 nonzeros N(0, 1/(d*d_model)), W2 nonzeros N(0, 2/(d*d_ff)).
    X0 [d_model x T] and targets [d_model x T] ~ N(0,1).
    """
    g = rng(seed)
    layers = []
    for _ in range(blocks):
        m1 = bernoulli_mask(g, d_ff, d_model, density)
        w1 = normal(g, (d_ff, d_model), 1.0 / (density * d_model))
        m2 = bernoulli_mask(g, d_model, d_ff, density)
        w2 = normal(g, (d_model, d_ff), 2.0 / (density * d_ff))
        layers.append((w1, m1, w2, m2))
    out = dict(layers=layers, blocks=blocks, d_model=d_model, d_ff=d_ff, T=T)
    if with_data:
        out["X0"] = normal(g, (d_model, T), 1.0)
        out["target"] = normal(g, (d_model, T), 1.0)
    return out


def token_shard(T: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous token range of `rank`: [r*T/G, (r+1)*T/G)."""
    base, extra = divmod(T, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)

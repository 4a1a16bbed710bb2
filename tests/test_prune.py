"""GMP schedule and magnitude pruning (§4.2.2, P559-P560; SPEC S404-S437
examples), host logic on CPU tensors."""
import math

import pytest
import torch

from paper_2302_04852_b200.prune import global_magnitude_masks, gmp_target_at, magnitude_mask


def test_gmp_schedule_examples_and_monotone():
    assert gmp_target_at(5, 0.95) == 0.0                      # dense for ten epochs
    assert gmp_target_at(10, 0.95) == pytest.approx(0.05)     # "pruning the lowest 5%" (P559)
    assert gmp_target_at(80, 0.95) == pytest.approx(0.95)
    assert gmp_target_at(100, 0.95) == pytest.approx(0.95)    # fine-tune: constant
    assert gmp_target_at(15, 0.95) == gmp_target_at(10, 0.95)  # held between pruning epochs
    seq = [gmp_target_at(e, 0.9) for e in range(0, 101)]
    assert all(b >= a for a, b in zip(seq, seq[1:]))


def test_magnitude_mask_examples():
    keep = magnitude_mask(torch.tensor([3.0, -1.0, 2.0, 0.5]), 0.5)
    assert keep.tolist() == [True, False, True, False]
    assert magnitude_mask(torch.randn(7, 5), 0.0).all()
    w = torch.randn(40, 30, generator=torch.Generator().manual_seed(0))
    k = magnitude_mask(w, 0.9)
    assert int(k.sum()) == math.ceil(0.1 * w.numel())
    assert w.abs()[k].min() >= w.abs()[~k].max()


def test_ties_keep_smaller_index():
    keep = magnitude_mask(torch.tensor([1.0, 1.0, 1.0, 1.0]), 0.5)
    assert keep.tolist() == [True, True, False, False]


def test_global_prunes_the_small_layer_first():
    a, b = torch.tensor([10.0, 10.0]), torch.tensor([0.1, 0.1])
    ka, kb = global_magnitude_masks([a, b], 0.5)
    assert ka.all() and not kb.any()


def test_pruning_within_current_mask_is_nested():
    w = torch.randn(50, 50, generator=torch.Generator().manual_seed(1))
    m1 = magnitude_mask(w, 0.8)
    m2 = magnitude_mask(w * m1, 0.95, current=m1)
    assert not (m2 & ~m1).any()
    assert int(m2.sum()) == 125

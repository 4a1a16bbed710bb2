"""The §4.2 dense/sparse dispatcher rule (P427-P429), host logic only."""
from paper_2302_04852_b200.nn import DENSE_BELOW, decide


def test_below_80_percent_is_dense_without_probing():
    calls = []
    t = lambda name: (lambda: calls.append(name) or 1.0)
    assert decide(0.5, t("dense"), t("sparse")) == "dense"
    assert decide(DENSE_BELOW - 1e-9, t("dense"), t("sparse")) == "dense"
    assert calls == []


def test_at_or_above_80_percent_the_faster_wins():
    assert decide(0.9, lambda: 2.0, lambda: 1.0) == "sparse"
    assert decide(0.99, lambda: 1.0, lambda: 3.0) == "dense"
    assert decide(DENSE_BELOW, lambda: 1.0, lambda: 1.0) == "sparse"   # tie -> sparse


def test_forced_modes():
    boom = lambda: (_ for _ in ()).throw(AssertionError("no probe in forced mode"))
    assert decide(0.1, boom, boom, mode="sparse") == "sparse"
    assert decide(0.99, boom, boom, mode="dense") == "dense"


def test_conv_considers_both_sparse_implementations():
    """P427: for convolution both sparse kernels (batch-last and OverON) are timed."""
    calls = []
    t = lambda name, v: (lambda: calls.append(name) or v)
    assert decide(0.9, t("dense", 3.0), t("sparse", 2.0), more_sparse={"sparse_nchw": t("nchw", 1.0)}) == "sparse_nchw"
    assert sorted(calls) == ["dense", "nchw", "sparse"]
    assert decide(0.9, lambda: 3.0, lambda: 1.0, more_sparse={"sparse_nchw": lambda: 2.0}) == "sparse"
    assert decide(0.9, lambda: 0.5, lambda: 1.0, more_sparse={"sparse_nchw": lambda: 2.0}) == "dense"
    assert decide(0.9, lambda: 1.0, lambda: 1.0, more_sparse={"sparse_nchw": lambda: 1.0}) == "sparse"  # ties
    assert decide(0.5, lambda: 1.0, lambda: 1.0, mode="sparse_nchw", more_sparse={"sparse_nchw": None}) == "sparse_nchw"

"""Pins of the LCN oracle (SPEC.md:215-223 examples; R15)."""
import numpy as np
import pytest

from oracle import lcn


def test_constant_and_zero_maps_give_zero():
    assert np.all(lcn(np.full((2, 9, 9, 3), 3.5), window=5) == 0)
    assert np.all(lcn(np.zeros((1, 7, 7, 2)), window=3) == 0)


def test_positive_scale_invariance():
    # lcn(c x) == lcn(x) within 1e-9 when the local std stays above the floor
    x = np.random.default_rng(0).standard_normal((2, 11, 10, 3))
    assert np.abs(lcn(7.0 * x, window=5) - lcn(x, window=5)).max() <= 1e-9


def test_hand_computed_1d_case():
    # one row of 3 pixels, window 3 (count-correct edges): means (1.5, 2, 2.5) for x = (1, 2, 3)
    x = np.array([1.0, 2.0, 3.0]).reshape(1, 1, 3, 1)
    with pytest.raises(ValueError):
        lcn(x, window=3)                                                     # window taller than the map
    x3 = np.repeat(x, 3, axis=1)                                             # 3 x 3 map, rows identical
    v = np.array([1 - 1.5, 2 - 2.0, 3 - 2.5])
    sd = np.sqrt(np.array([(v[0] ** 2 + v[1] ** 2) / 2, (v ** 2).sum() / 3, (v[1] ** 2 + v[2] ** 2) / 2]))
    want = v / np.maximum(1e-4, sd)
    got = lcn(x3, window=3)
    assert np.abs(got[0, 1, :, 0] - want).max() <= 1e-12
    assert np.abs(got[0, 0, :, 0] - want).max() <= 1e-12                   # columns see identical rows


def test_mirror_equivariance_and_channel_independence():
    x = np.random.default_rng(1).standard_normal((1, 8, 9, 2))
    y = lcn(x, window=5)
    assert np.abs(lcn(x[:, ::-1, ::-1, :], window=5) - y[:, ::-1, ::-1, :]).max() <= 1e-12
    x2 = x.copy()
    x2[..., 1] *= 3.0
    assert np.abs(lcn(x2, window=5)[..., 0] - y[..., 0]).max() == 0.0

"""Pins of the sparse-filter convolution and decide_format oracles:
a hand-computed example, equality with the (pinned) dense convolution of the densified
filter on several shapes, duplicate-column summing, an all-zero filter, the S:93-95
decide_format examples and idempotence."""
import numpy as np
import pytest

import oracle
import synth


def test_hand_example():
    # 1 image 1 channel 3x3, one filter with a single non-zero at tap (1, 2) of a 2x3 kernel:
    # y[p, q] = 2 * x[p + 1, q + 2] for the valid 2x1 output
    x = np.arange(9, dtype=np.float64).reshape(1, 9)
    y = oracle.conv2d_fwd_csr_filter(x, [0, 1], [5], [2.0], 1, 1, 3, 3, 1, 2, 3)
    assert np.array_equal(y, [[2 * 5.0, 2 * 8.0]])


SHAPES = [  # N, C, H, W, K, R, S, stride, pad, density
    (2, 1, 28, 28, 32, 5, 5, 1, 2, 0.3),
    (3, 4, 9, 7, 6, 3, 3, 2, 1, 0.5),
    (2, 3, 8, 8, 5, 1, 1, 1, 0, 0.2),
    (1, 2, 6, 5, 3, 4, 2, 1, (2, 0), 1.0),
]


@pytest.mark.parametrize("shape", SHAPES)
def test_equals_dense_conv_of_densified_filter(shape):
    N, C, H, W, K, R, S, st, pd, dens = shape
    pd = pd if isinstance(pd, tuple) else (pd, pd)
    rng = np.random.default_rng(7)
    x = rng.normal(size=(N, C * H * W))
    f = rng.normal(size=(K, C * R * S))
    f[rng.random(f.shape) > dens] = 0.0
    f[0] = 0.0                                  # an empty filter row
    f = f.astype(np.float32).astype(np.float64)  # to_csr stores float32 values
    rp, ci, v = synth.to_csr(f)
    b = rng.normal(size=K)
    y = oracle.conv2d_fwd_csr_filter(x, rp, ci, v, N, C, H, W, K, R, S, (st, st), pd, bias=b)
    yd = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S, (st, st), pd, bias=b)
    assert np.allclose(y, yd, rtol=0, atol=1e-12)


def test_duplicate_columns_are_summed():
    x = np.random.default_rng(1).normal(size=(1, 16))
    y1 = oracle.conv2d_fwd_csr_filter(x, [0, 2], [3, 3], [0.5, 0.25], 1, 1, 4, 4, 1, 2, 2)
    y2 = oracle.conv2d_fwd_csr_filter(x, [0, 1], [3], [0.75], 1, 1, 4, 4, 1, 2, 2)
    assert np.allclose(y1, y2, rtol=0, atol=1e-15)


def test_all_zero_filter_gives_bias():
    x = np.ones((2, 25))
    y = oracle.conv2d_fwd_csr_filter(x, [0, 0, 0], [], [], 2, 1, 5, 5, 2, 3, 3, bias=[1.5, -2.0])
    assert np.array_equal(y, np.repeat([[1.5] * 9 + [-2.0] * 9], 2, axis=0))


def test_decide_format_spec_examples():
    a = np.zeros((10, 10))
    a.flat[[3, 17, 42, 58, 99]] = 1.0                 # S:93 nnz = 5 -> sparse
    assert oracle.decide_format(a) == ("sparse", 5)
    assert oracle.decide_format(np.ones((10, 10))) == ("dense", 100)
    b = np.zeros((10, 10)); b.flat[:40] = 2.0          # exactly at the threshold -> sparse
    assert oracle.decide_format(b)[0] == "sparse"
    b.flat[40] = 2.0
    assert oracle.decide_format(b)[0] == "dense"
    # S:95 idempotence: densify(to_csr(a)) reproduces a bit-exactly, same decision
    rp, ci, v = synth.to_csr(a)
    a2 = oracle.csr_densify(rp, ci, v, 10, 10)
    assert np.array_equal(a2, a) and oracle.decide_format(a2) == oracle.decide_format(a)
    assert oracle.decide_format(np.array([[0.0, -0.0]]))[1] == 0  # signed zeros are not stored

"""Pins for the fp64 oracle's conv2d / bias / bwd_filter / bwd_data (CPU only).

Each test pins the oracle to something other than itself:
worked examples from SPEC.md (tests/golden), the im2col.GEMM identity
with an im2col helper that is itself pinned by the S:154 golden matrix, torch fp64
library routines, the adjoint identity (BJ north_star), central finite differences
 and linearity over samples.
"""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

import oracle
from tests.conftest import golden


def im2col(xrow, C, H, W, R, S, sh, sw, ph, pw):
    """Patch matrix (C*R*S) x (P*Q) by direct patch enumeration."""
    P = (H + 2 * ph - R) // sh + 1
    Q = (W + 2 * pw - S) // sw + 1
    x = np.asarray(xrow, dtype=np.float64).reshape(C, H, W)
    xp = np.zeros((C, H + 2 * ph, W + 2 * pw))
    xp[:, ph:ph + H, pw:pw + W] = x
    cols = np.empty((C * R * S, P * Q))
    for p in range(P):
        for q in range(Q):
            patch = xp[:, p * sh:p * sh + R, q * sw:q * sw + S]
            cols[:, p * Q + q] = patch.reshape(-1)
    return cols


def test_im2col_helper_matches_S154():
    g = golden("S154_im2col.txt")
    cols = im2col(g["x"], 1, 3, 3, 2, 2, 1, 1, 0, 0)
    for j in range(4):
        np.testing.assert_array_equal(cols[:, j], g[f"col{j}"])


@pytest.mark.parametrize("name", ["S163_conv.txt", "asym_conv.txt"])
def test_conv_worked_examples(name):
    g = golden(name)
    y = oracle.conv2d_fwd(np.array([g["x"]]), np.array([g["f"]]), 1, 1, 3, 3, 1, 2, 2)
    np.testing.assert_array_equal(y[0], g["y"])


def test_conv_identity_1x1():
    # S:162 "single 1x1 filter of value 1, C=1 -> output equals input"
    x = np.random.default_rng(0).uniform(-1, 1, size=(3, 1 * 5 * 7))
    y = oracle.conv2d_fwd(x, np.ones((1, 1)), 3, 1, 5, 7, 1, 1, 1)
    np.testing.assert_array_equal(y, x)


SHAPES = [
    # N, C, H, W, K, R, S, sh, sw, ph, pw
    (2, 3, 7, 6, 4, 3, 3, 1, 1, 1, 1),
    (2, 2, 9, 8, 3, 3, 2, 2, 2, 1, 0),
    (1, 3, 8, 8, 2, 5, 5, 1, 1, 2, 2),
    (2, 1, 6, 9, 3, 2, 3, 2, 1, 0, 1),
    (1, 4, 5, 5, 3, 1, 1, 1, 1, 0, 0),
    (2, 2, 7, 7, 2, 3, 3, 3, 2, 1, 1),  # floor extent: (7+2-3)/3+1 = 3
]


@pytest.mark.parametrize("shp", SHAPES)
def test_conv_fwd_equals_im2col_gemm(shp):
    N, C, H, W, K, R, S, sh, sw, ph, pw = shp
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, size=(N, C * H * W))
    f = rng.normal(size=(K, C * R * S))
    b = rng.normal(size=(K,))
    y = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S, (sh, sw), (ph, pw), bias=b)
    for n in range(N):
        ref = f @ im2col(x[n], C, H, W, R, S, sh, sw, ph, pw) + b[:, None]
        np.testing.assert_allclose(y[n], ref.reshape(-1), rtol=0, atol=1e-12)


@pytest.mark.parametrize("shp", SHAPES)
def test_conv_against_torch_fp64(shp):
    N, C, H, W, K, R, S, sh, sw, ph, pw = shp
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, size=(N, C * H * W))
    f = rng.normal(size=(K, C * R * S))
    b = rng.normal(size=(K,))
    dy_shape = None
    tx = torch.tensor(x).reshape(N, C, H, W)
    tf = torch.tensor(f).reshape(K, C, R, S)
    ty = Fn.conv2d(tx, tf, torch.tensor(b), stride=(sh, sw), padding=(ph, pw))
    y = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S, (sh, sw), (ph, pw), bias=b)
    np.testing.assert_allclose(y, ty.reshape(N, -1).numpy(), rtol=0, atol=1e-12)
    dy = rng.normal(size=ty.shape)
    tdy = torch.tensor(dy)
    gw = torch.nn.grad.conv2d_weight(tx, tf.shape, tdy, stride=(sh, sw), padding=(ph, pw))
    gx = torch.nn.grad.conv2d_input(tx.shape, tf, tdy, stride=(sh, sw), padding=(ph, pw))
    df, db = oracle.conv2d_bwd_filter(x, dy.reshape(N, -1), N, C, H, W, K, R, S, (sh, sw), (ph, pw))
    dx = oracle.conv2d_bwd_data(f, dy.reshape(N, -1), N, C, H, W, K, R, S, (sh, sw), (ph, pw))
    np.testing.assert_allclose(df, gw.reshape(K, -1).numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(dx, gx.reshape(N, -1).numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(db, tdy.sum(dim=(0, 2, 3)).numpy(), rtol=0, atol=1e-11)


@pytest.mark.parametrize("shp", SHAPES)
def test_adjoint_identity(shp):
    # BJ north_star: <conv(X,W),Y> = <X, conv_bwd_data(W,Y)> = <W, conv_bwd_filter(X,Y)>
    N, C, H, W, K, R, S, sh, sw, ph, pw = shp
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, size=(N, C * H * W))
    f = rng.normal(size=(K, C * R * S))
    y = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S, (sh, sw), (ph, pw))
    d = rng.normal(size=y.shape)
    dx = oracle.conv2d_bwd_data(f, d, N, C, H, W, K, R, S, (sh, sw), (ph, pw))
    df, _ = oracle.conv2d_bwd_filter(x, d, N, C, H, W, K, R, S, (sh, sw), (ph, pw))
    a = np.sum(y * d)
    assert abs(a - np.sum(x * dx)) <= 1e-12 * max(1.0, abs(a))
    assert abs(a - np.sum(f * df)) <= 1e-12 * max(1.0, abs(a))


def test_finite_differences_filter_data_bias():
    # S:172 / S:181: central differences h = 1e-5, relative error <= 1e-6
    N, C, H, W, K, R, S, sh, sw, ph, pw = (2, 2, 5, 6, 3, 3, 3, 2, 1, 1, 1)
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, size=(N, C * H * W))
    f = rng.normal(size=(K, C * R * S))
    b = rng.normal(size=(K,))
    y = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S, (sh, sw), (ph, pw), bias=b)
    d = rng.normal(size=y.shape)
    loss = lambda xx, ff, bb: np.sum(d * oracle.conv2d_fwd(xx, ff, N, C, H, W, K, R, S, (sh, sw), (ph, pw), bias=bb))
    df, db = oracle.conv2d_bwd_filter(x, d, N, C, H, W, K, R, S, (sh, sw), (ph, pw))
    dx = oracle.conv2d_bwd_data(f, d, N, C, H, W, K, R, S, (sh, sw), (ph, pw))
    h = 1e-5
    for i in rng.choice(f.size, 8, replace=False):
        fp, fm = f.copy(), f.copy()
        fp.flat[i] += h; fm.flat[i] -= h
        fd = (loss(x, fp, b) - loss(x, fm, b)) / (2 * h)
        assert abs(fd - df.flat[i]) <= 1e-6 * max(1.0, abs(fd))
    for i in rng.choice(x.size, 8, replace=False):
        xp_, xm = x.copy(), x.copy()
        xp_.flat[i] += h; xm.flat[i] -= h
        fd = (loss(xp_, f, b) - loss(xm, f, b)) / (2 * h)
        assert abs(fd - dx.flat[i]) <= 1e-6 * max(1.0, abs(fd))
    for k in range(K):
        bp, bm = b.copy(), b.copy()
        bp[k] += h; bm[k] -= h
        fd = (loss(x, f, bp) - loss(x, f, bm)) / (2 * h)
        assert abs(fd - db[k]) <= 1e-6 * max(1.0, abs(fd))


def test_linearity_and_zero_dout():
    # S:173 "N=2 gradient equals sum of the two N=1 gradients"; S:171/S:179 dout=0 -> 0
    C, H, W, K, R, S = 2, 6, 6, 3, 3, 3
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, size=(2, C * H * W))
    d = rng.normal(size=(2, K * 6 * 6))
    df2, db2 = oracle.conv2d_bwd_filter(x, d, 2, C, H, W, K, R, S, (1, 1), (1, 1))
    dfa, dba = oracle.conv2d_bwd_filter(x[:1], d[:1], 1, C, H, W, K, R, S, (1, 1), (1, 1))
    dfb, dbb = oracle.conv2d_bwd_filter(x[1:], d[1:], 1, C, H, W, K, R, S, (1, 1), (1, 1))
    np.testing.assert_allclose(df2, dfa + dfb, rtol=0, atol=1e-12)
    np.testing.assert_allclose(db2, dba + dbb, rtol=0, atol=1e-12)
    z = np.zeros_like(d)
    df0, db0 = oracle.conv2d_bwd_filter(x, z, 2, C, H, W, K, R, S, (1, 1), (1, 1))
    assert not df0.any() and not db0.any()
    dx0 = oracle.conv2d_bwd_data(rng.normal(size=(K, C * R * S)), z, 2, C, H, W, K, R, S, (1, 1), (1, 1))
    assert not dx0.any()


def test_bwd_data_identity_1x1():
    # S:180 "identity 1x1 filter -> dX == dout"
    d = np.random.default_rng(6).normal(size=(2, 1 * 4 * 5))
    dx = oracle.conv2d_bwd_data(np.ones((1, 1)), d, 2, 1, 4, 5, 1, 1, 1)
    np.testing.assert_array_equal(dx, d)


def test_bias_add_matches_conv_bias():
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, size=(2, 2 * 5 * 5))
    f = rng.normal(size=(3, 2 * 9))
    b = rng.normal(size=(3,))
    y0 = oracle.conv2d_fwd(x, f, 2, 2, 5, 5, 3, 3, 3, (1, 1), (1, 1))
    yb = oracle.conv2d_fwd(x, f, 2, 2, 5, 5, 3, 3, 3, (1, 1), (1, 1), bias=b)
    tx = torch.tensor(x).reshape(2, 2, 5, 5)
    ty = Fn.conv2d(tx, torch.tensor(f).reshape(3, 2, 3, 3), torch.tensor(b), padding=1)
    np.testing.assert_allclose(oracle.bias_add(y0, b, 2, 3, 25), ty.reshape(2, -1).numpy(), atol=1e-12, rtol=0)
    np.testing.assert_allclose(yb, ty.reshape(2, -1).numpy(), atol=1e-12, rtol=0)


def test_out_extent_floor_reading():
    # reading R2: floor; ResNet-50 stem 7x7/2 p3 on 224 -> 112 (SURVEY §8(c) ambiguity 2)
    assert oracle.out_extent(224, 3, 7, 2) == 112
    assert oracle.out_extent(28, 2, 5, 1) == 28
    assert oracle.out_extent(3, 0, 5, 1) == 0


def _sweep_shapes():
    out = []
    for N, C, K, H, W, R, S, st, pd in itertools.product(
            (1, 2), (1, 3), (1, 2), (1, 4, 6), (2, 5), (1, 2, 3), (1, 3), (1, 2), (0, 1)):
        if (H + 2 * pd - R) < 0 or (W + 2 * pd - S) < 0:
            continue
        out.append((N, C, H, W, K, R, S, st, st, pd, pd))
    return out


def test_bruteforce_sweep_im2col_identity():
    # S:202 / S:573: im2col path == direct loops within 1e-10 over small shapes
    # (a deterministic subsample of the N,C,K<=3, H,W<=6, kernel<=3, stride{1,2}, pad{0,1} grid)
    shapes = _sweep_shapes()
    rng = np.random.default_rng(8)
    for shp in shapes[::3]:
        N, C, H, W, K, R, S, sh, sw, ph, pw = shp
        x = rng.uniform(-1, 1, size=(N, C * H * W))
        f = rng.normal(size=(K, C * R * S))
        y = oracle.conv2d_fwd(x, f, N, C, H, W, K, R, S, (sh, sw), (ph, pw))
        for n in range(N):
            ref = (f @ im2col(x[n], C, H, W, R, S, sh, sw, ph, pw)).reshape(-1)
            assert np.max(np.abs(y[n] - ref), initial=0.0) <= 1e-10, shp


def test_csr_densify():
    # P:130-131 CSR; S:28-34 invariants.  Known 2x4 example + duplicate summing (reading R15)
    rp = np.array([0, 2, 3], dtype=np.int32)
    ci = np.array([1, 3, 0], dtype=np.int32)
    v = np.array([5.0, -1.0, 2.0])
    np.testing.assert_array_equal(oracle.csr_densify(rp, ci, v, 2, 4), [[0, 5, 0, -1], [2, 0, 0, 0]])
    np.testing.assert_array_equal(
        oracle.csr_densify(np.array([0, 2], np.int32), np.array([1, 1], np.int32), np.array([1.5, 2.0]), 1, 3),
        [[0, 3.5, 0]])
    import synth
    d = synth.mnist_like(16, seed=(99,))
    rp, ci, v = synth.to_csr(d)
    np.testing.assert_array_equal(oracle.csr_densify(rp, ci, v, 16, 784), d.astype(np.float64))

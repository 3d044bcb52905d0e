"""Pins for the fp64 oracle's relu_maxpool / maxpool_bwd / LeNet step / SGD (CPU only)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

import oracle
import synth
from tests.conftest import golden


def torch_pool(x, N, C, H, W, R, S, st, pd, relu=True):
    t = torch.tensor(np.asarray(x, dtype=np.float64)).reshape(N, C, H, W)
    if relu:
        t = torch.clamp(t, min=0.0)  # +0.0 for negatives (clamp keeps -0.0 only for -0.0 input)
    out, idx = Fn.max_pool2d(t, (R, S), stride=st, padding=pd, return_indices=True)
    P, Q = out.shape[2], out.shape[3]
    # torch returns h*W+w per plane; reading R6 adds the channel offset c*H*W
    idx = idx + (torch.arange(C) * H * W).reshape(1, C, 1, 1)
    return out.reshape(N, -1).numpy(), idx.reshape(N, -1).numpy().astype(np.int32), P, Q


def test_pool_S188_example():
    g = golden("S188_pool.txt")
    out, arg = oracle.relu_maxpool(np.array([g["x"]]), 1, 1, 2, 2, 2, 2, (2, 2), (0, 0), relu=False)
    assert out[0, 0] == g["out"][0] and arg[0, 0] == int(g["argmax"][0])


def test_pool_constant_input_first_index_and_1x1_identity():
    # S:189 constant input -> constant output, argmax = first index per window (reading R5)
    x = np.full((1, 1 * 4 * 4), 2.5)
    out, arg = oracle.relu_maxpool(x, 1, 1, 4, 4, 2, 2, (2, 2), (0, 0))
    np.testing.assert_array_equal(out, 2.5)
    np.testing.assert_array_equal(arg[0], [0, 2, 8, 10])
    # S:190 window 1x1 stride 1 -> identity
    x = np.random.default_rng(0).uniform(-1, 1, size=(2, 3 * 3 * 4))
    out, arg = oracle.relu_maxpool(x, 2, 3, 3, 4, 1, 1, (1, 1), (0, 0), relu=False)
    np.testing.assert_array_equal(out, x)
    np.testing.assert_array_equal(arg, np.tile(np.arange(36), (2, 1)))


@pytest.mark.parametrize("cfg", [
    # N, C, H, W, R, S, st, pd
    (2, 3, 8, 8, 2, 2, 2, 0),
    (2, 2, 7, 9, 3, 3, 2, 1),
    (1, 4, 6, 6, 3, 3, 1, 1),
    (2, 2, 5, 7, 2, 3, (1, 2), (1, 1)),
])
@pytest.mark.parametrize("relu", [True, False])
def test_pool_against_torch_ties_included(cfg, relu):
    N, C, H, W, R, S, st, pd = cfg
    st = st if isinstance(st, tuple) else (st, st)
    pd = pd if isinstance(pd, tuple) else (pd, pd)
    rng = np.random.default_rng(1)
    for data in (rng.uniform(-1, 1, size=(N, C * H * W)),
                 rng.integers(-1, 2, size=(N, C * H * W)).astype(np.float64)):  # heavy ties
        out, arg = oracle.relu_maxpool(data, N, C, H, W, R, S, st, pd, relu=relu)
        tout, targ, P, Q = torch_pool(data, N, C, H, W, R, S, st, pd, relu=relu)
        np.testing.assert_array_equal(out, tout)
        np.testing.assert_array_equal(arg, targ)


def test_maxpool_bwd_against_torch_autograd():
    # route dout to argmax, collisions summed; with relu mask (reading R9) this
    # equals relu_backward(maxpool_backward(relu x)), i.e. torch autograd of maxpool(relu(x))
    N, C, H, W, R, S = 2, 3, 7, 7, 3, 3
    st, pd = (2, 2), (1, 1)  # overlapping windows -> collisions
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, size=(N, C * H * W))
    for relu in (False, True):
        t = torch.tensor(x).reshape(N, C, H, W).requires_grad_(True)
        y = Fn.max_pool2d(torch.relu(t) if relu else t, (R, S), stride=st, padding=pd)
        dout = rng.normal(size=y.shape)
        y.backward(torch.tensor(dout))
        out, arg = oracle.relu_maxpool(x, N, C, H, W, R, S, st, pd, relu=relu)
        P, Q = y.shape[2], y.shape[3]
        dx = oracle.maxpool_bwd(arg, dout.reshape(N, -1), N, C, H, W, P, Q,
                                out_mask=out if relu else None)
        np.testing.assert_allclose(dx, t.grad.reshape(N, -1).numpy(), rtol=0, atol=1e-14)


def test_maxpool_bwd_exact_when_stride_ge_window_and_fd():
    N, C, H, W = 2, 2, 6, 6
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, size=(N, C * H * W))
    out, arg = oracle.relu_maxpool(x, N, C, H, W, 2, 2, (2, 2), (0, 0), relu=False)
    dout = rng.normal(size=out.shape)
    dx = oracle.maxpool_bwd(arg, dout, N, C, H, W, 3, 3)
    # each dX element receives at most one term -> exactly dout at argmax, 0 elsewhere
    assert np.count_nonzero(dx) == dout.size
    for n in range(N):
        np.testing.assert_array_equal(dx[n, arg[n]], dout[n])
    # S:198 finite differences away from ties
    h = 1e-6
    for i in rng.choice(x.size, 10, replace=False):
        xp_, xm = x.copy(), x.copy()
        xp_.flat[i] += h; xm.flat[i] -= h
        fp = np.sum(dout * oracle.relu_maxpool(xp_, N, C, H, W, 2, 2, (2, 2), (0, 0), relu=False)[0])
        fm = np.sum(dout * oracle.relu_maxpool(xm, N, C, H, W, 2, 2, (2, 2), (0, 0), relu=False)[0])
        assert abs((fp - fm) / (2 * h) - dx.flat[i]) <= 1e-6


def test_fully_padded_window_reading_R4():
    # fully padded window -> output 0; argmax -1 (never routed)
    x = np.array([[5.0]])
    out, arg = oracle.relu_maxpool(x, 1, 1, 1, 1, 1, 1, (1, 1), (1, 1), relu=False)
    np.testing.assert_array_equal(out[0], [0, 0, 0, 0, 5, 0, 0, 0, 0])
    np.testing.assert_array_equal(arg[0], [-1, -1, -1, -1, 0, -1, -1, -1, -1])


# ---------------------------------------------------------------------------- LeNet

def torch_lenet(x, labels, params, n_global):
    p = synth.split_lenet_params(params.astype(np.float64))
    t = {k: torch.tensor(v, requires_grad=True) for k, v in p.items()}
    n = x.shape[0]
    X = torch.tensor(np.asarray(x, dtype=np.float64)).reshape(n, 1, 28, 28)
    z1 = Fn.conv2d(X, t["F1"].reshape(32, 1, 5, 5), t["b1"], padding=2)
    a1 = Fn.max_pool2d(torch.relu(z1), 2)
    z2 = Fn.conv2d(a1, t["F2"].reshape(64, 32, 5, 5), t["b2"], padding=2)
    a2 = Fn.max_pool2d(torch.relu(z2), 2).reshape(n, -1)
    s = a2 @ t["W3"].T + t["b3"]
    loss = Fn.cross_entropy(s, torch.tensor(labels, dtype=torch.long), reduction="sum") / n_global
    loss.backward()
    g = np.concatenate([t[k].grad.numpy().ravel() for k, _ in synth.LENET_PARAM_SHAPES])
    return g, loss.item()


def test_lenet_num_params():
    assert oracle.lenet_num_params() == synth.LENET_NUM_PARAMS == 83466


def test_lenet_step_against_torch_autograd():
    n = 3
    x = synth.mnist_like(n, seed=(10,))
    y = synth.labels(n, seed=(11,))
    prm = synth.lenet_params(seed=(12,))
    # non-zero biases so that every parameter block is exercised
    prm = prm + synth.normal(prm.shape, 0.01, seed=(13,))
    g, loss = oracle.lenet_fwd_bwd(x, y, prm, n_global=7)
    tg, tloss = torch_lenet(x, y, prm, 7)
    assert abs(loss - tloss) <= 1e-12
    np.testing.assert_allclose(g, tg, rtol=0, atol=1e-12 * max(1.0, np.abs(tg).max()))


def test_lenet_finite_differences():
    # S:274 / S:572 end-to-end gradient check through conv->relu->pool->affine
    n = 2
    x = synth.mnist_like(n, seed=(20,))
    y = synth.labels(n, seed=(21,))
    prm = (synth.lenet_params(seed=(22,)) + synth.normal((83466,), 0.01, seed=(23,))).astype(np.float64)
    g, _ = oracle.lenet_fwd_bwd(x, y, prm)
    rng = np.random.default_rng(24)
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in synth.LENET_PARAM_SHAPES])
    h = 1e-5
    for blk in range(6):
        for i in rng.integers(offs[blk], offs[blk + 1], size=3):
            pp, pm = prm.copy(), prm.copy()
            pp[i] += h; pm[i] -= h
            fd = (oracle.lenet_fwd_bwd(x, y, pp)[1] - oracle.lenet_fwd_bwd(x, y, pm)[1]) / (2 * h)
            assert abs(fd - g[i]) <= 1e-5 * max(1e-3, abs(fd)), (blk, i, fd, g[i])


def test_lenet_uniform_logits_loss_ln10_and_p_minus_y():
    # S:253 uniform logits; "uniform probs over K -> loss = ln K"; S:259 ds = p - y
    n = 4
    x = synth.mnist_like(n, seed=(30,))
    y = synth.labels(n, seed=(31,))
    prm = synth.lenet_params(seed=(32,)).astype(np.float64)
    prm[-(31360 + 10):] = 0.0  # W3 = 0, b3 = 0 -> scores 0 -> p = 1/10
    g, loss = oracle.lenet_fwd_bwd(x, y, prm)
    assert abs(loss - np.log(10.0)) <= 1e-14
    db3 = g[-10:]
    onehot = np.eye(10)[y]
    np.testing.assert_allclose(db3, (0.1 - onehot).sum(0) / n, rtol=0, atol=1e-15)


def test_data_parallel_shard_sum_equals_full_batch():
    # S:499 "concat-data grad = sum of partition grads" (the DP allreduce reading, §8(e))
    n = 4
    x = synth.mnist_like(n, seed=(40,))
    y = synth.labels(n, seed=(41,))
    prm = synth.lenet_params(seed=(42,))
    g, loss = oracle.lenet_fwd_bwd(x, y, prm, n_global=n)
    ga, la = oracle.lenet_fwd_bwd(x[:2], y[:2], prm, n_global=n)
    gb, lb = oracle.lenet_fwd_bwd(x[2:], y[2:], prm, n_global=n)
    np.testing.assert_allclose(g, ga + gb, rtol=0, atol=1e-15)
    assert abs(loss - (la + lb)) <= 1e-14


def test_sgd_S288():
    g = golden("S288_sgd.txt")
    out = oracle.sgd_update(np.array(g["p"]), np.array(g["g"]), g["lr"][0])
    assert abs(out[0] - g["out"][0]) <= 1e-16


def test_dyadic_lenet_forward_is_exact_in_fp32():
    # The family-G LeNet grid makes conv1/conv2 + bias exact in fp32:
    # check the fp64 oracle's pooled activations are representable in fp32 exactly.
    x = synth.mnist_like_dyadic(4)
    prm = synth.lenet_params(dyadic_grid=True)
    fw = oracle.lenet_forward(x, prm)
    for k in ("a1", "a2"):
        assert np.array_equal(fw[k].astype(np.float32).astype(np.float64), fw[k])


def test_lenet_predict_properties():
    """Scoring oracle: probabilities sum to 1, the label is the argmax of the
    (pinned) forward scores, and a common shift of the logits (added to every b3 entry)
    leaves the probabilities unchanged (softmax shift invariance)."""
    rng = np.random.default_rng(5)
    x = rng.random((6, 784))
    prm = synth.lenet_params(seed=(31,)).astype(np.float64)
    pred, probs = oracle.lenet_predict(x, prm)
    assert np.allclose(probs.sum(axis=1), 1.0, rtol=0, atol=1e-14)
    assert np.array_equal(pred, np.argmax(oracle.lenet_forward(x, prm)["scores"], axis=1))
    prm2 = prm.copy()
    prm2[-10:] += 3.25
    assert np.allclose(oracle.lenet_predict(x, prm2)[1], probs, rtol=0, atol=1e-12)


def test_lenet_predict_vs_torch_softmax_fp64():
    """oracle_lenet_predict's softmax against torch.softmax in fp64 on the
    oracle's own forward scores (pinned above), and its label against torch.argmax
    (first maximal index).  A base-2 exponential, a missing max shift that overflows, or a
    wrong normalisation axis fails here."""
    import torch
    rng = np.random.default_rng(7)
    x = rng.random((9, 784))
    prm = synth.lenet_params(seed=(33,)).astype(np.float64)
    prm[-10:] += rng.normal(0, 3.0, 10)        # spread the logits so the softmax is not flat
    sc = torch.from_numpy(oracle.lenet_forward(x, prm)["scores"])
    pred, probs = oracle.lenet_predict(x, prm)
    ref = torch.softmax(sc, dim=1).numpy()
    assert np.abs(probs - ref).max() <= 1e-14
    assert np.array_equal(pred, torch.argmax(sc, dim=1).numpy().astype(np.int32))


def test_lenet_predict_closed_forms():
    """Closed forms of the scoring softmax: W3 = 0 makes the logits equal b3 for every image.
    b3 = 0 -> p = 1/10 and label 0 (first maximal class of a ten-way tie);
    b3 = (ln 2, 0, ..., 0) -> p0 = 2/11, pj = 1/11; b3 = 800 on class 7 only -> label 7, p7 ~ 1
    without overflow (the max shift)."""
    x = synth.mnist_like(3, seed=(34,)).astype(np.float64)
    prm = synth.lenet_params(seed=(35,)).astype(np.float64)
    prm[-10 - 31360:-10] = 0.0
    prm[-10:] = 0.0
    pred, probs = oracle.lenet_predict(x, prm)
    assert np.array_equal(pred, [0, 0, 0]) and np.abs(probs - 0.1).max() <= 1e-15
    prm[-10] = np.log(2.0)
    pred, probs = oracle.lenet_predict(x, prm)
    assert np.abs(probs[:, 0] - 2 / 11).max() <= 1e-15 and np.abs(probs[:, 1:] - 1 / 11).max() <= 1e-15
    prm[-10:] = 0.0
    prm[-3] = 800.0
    pred, probs = oracle.lenet_predict(x, prm)
    assert np.array_equal(pred, [7, 7, 7]) and np.all(np.isfinite(probs))
    assert np.abs(probs[:, 7] - 1.0).max() <= 1e-15

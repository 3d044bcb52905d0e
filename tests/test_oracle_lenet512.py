"""Pins for the oracle's NEXT-4 functions (CPU only): the Philox4x64-10 generator, inverted
dropout, and the LeNet-512 step (SystemML mnist_lenet topology, R22-R24).

Each pin is independent of the oracle's own arithmetic: numpy's Philox (a library routine),
torch fp64 autograd of the same network, central finite differences, statistical laws of the
Bernoulli mask, closed forms (uniform logits), and the shard-sum identity."""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

import oracle
import synth

H = synth.LENET512_HIDDEN


def test_num_params():
    assert oracle.lenet512_num_params() == synth.LENET512_NUM_PARAMS == 1663370


@pytest.mark.parametrize("key", [0, 5, 180204647 + (3 << 64), 2**128 - 1])
def test_philox_matches_numpy(key):
    # library pin: numpy.random.Philox is Philox4x64-10 with the same counter convention
    ref = np.random.Philox(key=key).random_raw(40)
    k0, k1 = key & (2**64 - 1), key >> 64
    np.testing.assert_array_equal(oracle.philox_raw(k0, k1, 0, 40), ref)
    np.testing.assert_array_equal(oracle.philox_raw(k0, k1, 13, 27), ref[13:])


def test_dropout_mask_keep_one_rate_and_global_row_indexing():
    # S:279 example "keep_p = 1 -> out == x, mask all ones"
    assert oracle.dropout_mask(7, 3, 0, 16, H, 1.0).all()
    for keep in (0.5, 0.8, 0.1):
        m = oracle.dropout_mask(11, 2, 0, 2048, H, keep)
        n = m.size
        frac = m.mean()
        assert abs(frac - keep) <= 5 * np.sqrt(keep * (1 - keep) / n), (keep, frac)
    # the mask is a function of the GLOBAL sample row (any sharding draws the same mask)
    full = oracle.dropout_mask(5, 9, 0, 10, H, 0.5)
    np.testing.assert_array_equal(oracle.dropout_mask(5, 9, 3, 4, H, 0.5), full[3:7])
    # the definition: kept iff the high 32 bits of raw output (row*H + j) are < keep * 2^32
    raw = np.random.Philox(key=5 + (9 << 64)).random_raw(10 * H).reshape(10, H)
    np.testing.assert_array_equal(full, ((raw >> np.uint64(32)) < np.uint64(2**31)).astype(np.uint8))
    # different steps draw different masks (a stuck step counter would repeat them)
    assert (oracle.dropout_mask(5, 10, 0, 10, H, 0.5) != full).mean() > 0.4


def test_dropout_monte_carlo_mean():
    # S:278 "expectation check: mean over 10^4 seeded draws within 2% of x"
    D, draws, keep = 64, 10000, 0.5
    x = synth.uniform((D,), 0.5, 1.5, seed=(50,)).astype(np.float64)
    acc = np.zeros(D)
    masks = oracle.dropout_mask(123, 0, 0, draws, D, keep)  # row i = draw i
    for i in range(draws):
        acc += oracle.dropout_fwd(x, masks[i], keep)
    mean = acc / draws
    sigma = x * np.sqrt((1 - keep) / keep / draws)
    assert np.all(np.abs(mean - x) <= 5 * sigma)
    assert abs(mean.sum() - x.sum()) <= 0.02 * x.sum()


def test_dropout_backward_routes_only_kept_units_and_is_adjoint():
    x = synth.uniform((4, H), seed=(51,)).astype(np.float64)
    d = synth.uniform((4, H), seed=(52,)).astype(np.float64)
    m = oracle.dropout_mask(1, 1, 0, 4, H, 0.7)
    dx = oracle.dropout_bwd(d, m, 0.7)
    assert np.all(dx[m == 0] == 0.0)
    np.testing.assert_allclose(dx[m == 1], d[m == 1] / 0.7, rtol=1e-15)
    y = oracle.dropout_fwd(x, m, 0.7)
    assert abs((y * d).sum() - (x * dx).sum()) <= 1e-12   # <fwd(x), d> = <x, bwd(d)>
    np.testing.assert_array_equal(oracle.dropout_fwd(x, np.ones_like(m), 1.0), x)  # keep_p = 1


def torch_lenet512(x, labels, params, n_global, mask, keep):
    p = synth.split_lenet512_params(params.astype(np.float64))
    t = {k: torch.tensor(v, requires_grad=True) for k, v in p.items()}
    n = x.shape[0]
    X = torch.tensor(np.asarray(x, dtype=np.float64)).reshape(n, 1, 28, 28)
    z1 = Fn.conv2d(X, t["F1"].reshape(32, 1, 5, 5), t["b1"], padding=2)
    a1 = Fn.max_pool2d(torch.relu(z1), 2)
    z2 = Fn.conv2d(a1, t["F2"].reshape(64, 32, 5, 5), t["b2"], padding=2)
    a2 = Fn.max_pool2d(torch.relu(z2), 2).reshape(n, -1)
    z3 = a2 @ t["W3"].T + t["b3"]
    h = torch.relu(z3) * torch.tensor(mask, dtype=torch.float64) / keep
    s = h @ t["W4"].T + t["b4"]
    loss = Fn.cross_entropy(s, torch.tensor(labels, dtype=torch.long), reduction="sum") / n_global
    loss.backward()
    g = np.concatenate([t[k].grad.numpy().ravel() for k, _ in synth.LENET512_PARAM_SHAPES])
    return g, loss.item(), s.detach().numpy()


def _noisy_params(seed):
    prm = synth.lenet512_params(seed=seed).astype(np.float64)
    return prm + synth.normal(prm.shape, 0.01, seed=seed + (1,))


def test_lenet512_against_torch_autograd():
    n, keep, seed, step = 3, 0.5, 77, 4
    x = synth.mnist_like(n, seed=(60,))
    y = synth.labels(n, seed=(61,))
    prm = _noisy_params((62,))
    row0 = 5
    g, loss = oracle.lenet512_fwd_bwd(x, y, prm, seed, step, keep, n_global=7, row0=row0)
    mask = oracle.dropout_mask(seed, step, row0, n, H, keep)
    assert 0 < mask.mean() < 1
    tg, tloss, _ = torch_lenet512(x, y, prm, 7, mask, keep)
    assert abs(loss - tloss) <= 1e-12
    np.testing.assert_allclose(g, tg, rtol=0, atol=1e-12 * max(1.0, np.abs(tg).max()))
    fw = oracle.lenet512_forward(x, prm, train=True, seed=seed, step=step, keep_p=keep, row0=row0)
    np.testing.assert_array_equal(fw["mask"], mask)


def test_lenet512_finite_differences():
    # S:274 end-to-end gradient check (the mask is fixed by (seed, step, row))
    n, keep, seed, step = 2, 0.6, 3, 1
    x = synth.mnist_like(n, seed=(63,))
    y = synth.labels(n, seed=(64,))
    prm = _noisy_params((65,))
    g, _ = oracle.lenet512_fwd_bwd(x, y, prm, seed, step, keep)
    rng = np.random.default_rng(66)
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in synth.LENET512_PARAM_SHAPES])
    h = 1e-5
    for blk in range(8):
        idx = rng.integers(offs[blk], offs[blk + 1], size=2)
        if blk == 4:  # W3: also probe the largest-gradient entry (most W3 entries are ~0)
            idx = np.append(idx, offs[4] + np.argmax(np.abs(g[offs[4]:offs[5]])))
        for i in idx:
            pp, pm = prm.copy(), prm.copy()
            pp[i] += h; pm[i] -= h
            fd = (oracle.lenet512_fwd_bwd(x, y, pp, seed, step, keep)[1]
                  - oracle.lenet512_fwd_bwd(x, y, pm, seed, step, keep)[1]) / (2 * h)
            assert abs(fd - g[i]) <= 1e-5 * max(1e-3, abs(fd)), (blk, i, fd, g[i])


def test_lenet512_uniform_logits_closed_form():
    # W4 = 0, b4 = 0: scores 0 -> p = 1/10, loss = ln 10, db4 = sum (p - y)/N,
    # and dh = ds W4 = 0, so every gradient below the output layer is exactly 0.
    n = 4
    x = synth.mnist_like(n, seed=(67,))
    y = synth.labels(n, seed=(68,))
    prm = _noisy_params((69,))
    prm[-(10 * H + 10):] = 0.0
    g, loss = oracle.lenet512_fwd_bwd(x, y, prm, 1, 1, 0.5)
    assert abs(loss - np.log(10.0)) <= 1e-14
    np.testing.assert_allclose(g[-10:], (0.1 - np.eye(10)[y]).sum(0) / n, rtol=0, atol=1e-15)
    assert np.all(g[:-(10 * H + 10)] == 0.0)


def test_lenet512_shard_sum_equals_full_batch():
    # S:499, with the mask indexed by the global row: shards [0,2) and [2,5) of one batch
    n, keep = 5, 0.5
    x = synth.mnist_like(n, seed=(70,))
    y = synth.labels(n, seed=(71,))
    prm = _noisy_params((72,))
    g, loss = oracle.lenet512_fwd_bwd(x, y, prm, 9, 2, keep, n_global=n)
    ga, la = oracle.lenet512_fwd_bwd(x[:2], y[:2], prm, 9, 2, keep, n_global=n, row0=0)
    gb, lb = oracle.lenet512_fwd_bwd(x[2:], y[2:], prm, 9, 2, keep, n_global=n, row0=2)
    np.testing.assert_allclose(g, ga + gb, rtol=0, atol=1e-15)
    assert abs(loss - (la + lb)) <= 1e-14


def test_lenet512_predict_vs_torch_softmax():
    n = 6
    x = synth.mnist_like(n, seed=(73,))
    prm = _noisy_params((74,))
    pred, probs = oracle.lenet512_predict(x, prm)
    _, _, s = torch_lenet512(x, np.zeros(n, np.int32), prm, n, np.ones((n, H), np.uint8), 1.0)
    np.testing.assert_allclose(probs, torch.softmax(torch.tensor(s), 1).numpy(), rtol=0, atol=1e-14)
    np.testing.assert_array_equal(pred, np.argmax(s, axis=1))
    # scoring uses no dropout: keep_p = 1 training forward gives the same scores
    fw = oracle.lenet512_forward(x, prm, train=True, seed=1, step=1, keep_p=1.0)
    np.testing.assert_allclose(fw["scores"], s, rtol=0, atol=1e-12)

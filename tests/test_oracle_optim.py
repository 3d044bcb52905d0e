"""Pins of the optimizer oracle (oracle_optimizer_update; P:49 six optimizers)
against closed forms derived independently of the update recurrences, the worked example
S:290 gives, special cases that reduce to plain SGD, and the zero-gradient invariant S:289."""
import numpy as np
import pytest

import oracle

KINDS = ["sgd", "momentum", "nesterov", "adagrad", "rmsprop", "adam"]


def run(kind, p0, g, steps, **hp):
    p = np.array(p0, dtype=np.float64)
    st = np.zeros(oracle.OPT_STATE[kind] * p.size)
    for t in range(1, steps + 1):
        p, st = oracle.optimizer_update(kind, p, g, st, t=t, **hp)
    return p, st


@pytest.mark.parametrize("kind", KINDS)
def test_zero_gradient_leaves_params(kind):
    # g = 0 with zero accumulators -> parameters unchanged
    p0 = np.linspace(-2, 3, 17)
    p, st = run(kind, p0, np.zeros(17), 4)
    assert np.array_equal(p, p0)
    assert not np.any(st)


def test_adam_worked_example():
    # adam step 1 on p = 0, g = 1 -> p = -lr * 1 / (sqrt(1) + eps) (corrections cancel)
    lr, eps = 0.01, 1e-8
    p, st = oracle.optimizer_update("adam", np.zeros(1), np.ones(1), np.zeros(2), t=1, lr=lr, eps=eps)
    assert abs(p[0] - (-lr / (1.0 + eps))) <= 1e-17
    assert np.allclose(st, [0.1, 0.001], rtol=0, atol=1e-15)


@pytest.mark.parametrize("kind", ["momentum", "nesterov"])
def test_mu_zero_is_sgd(kind):
    rng = np.random.default_rng(3)
    p0, g = rng.normal(size=50), rng.normal(size=50)
    p_sgd, _ = oracle.optimizer_update("sgd", p0, g, np.zeros(0), lr=0.05)
    p, _ = oracle.optimizer_update(kind, p0, g, np.zeros(50), lr=0.05, mu=0.0)
    assert np.array_equal(p, p_sgd)


def test_momentum_constant_gradient_closed_form():
    # v_k = -lr g (1 - mu^k) / (1 - mu);  p_k = p_0 + sum_i v_i (geometric series)
    lr, mu, k = 0.01, 0.9, 12
    g = np.array([1.5, -0.25, 3.0])
    p, v = run("momentum", np.zeros(3), g, k, lr=lr, mu=mu)
    vk = -lr * g * (1 - mu ** k) / (1 - mu)
    pk = -lr * g / (1 - mu) * (k - mu * (1 - mu ** k) / (1 - mu))
    assert np.allclose(v, vk, rtol=1e-13, atol=0)
    assert np.allclose(p, pk, rtol=1e-13, atol=0)


def test_nesterov_telescopes_to_momentum_plus_mu_v():
    # p_k - p_{k-1} = v_k + mu (v_k - v_{k-1}) telescopes to p_k = p_0 + sum_i v_i + mu v_k
    lr, mu, k = 0.02, 0.8, 9
    g = np.array([0.7, -1.1])
    p_m, v_m = run("momentum", np.zeros(2), g, k, lr=lr, mu=mu)
    p_n, v_n = run("nesterov", np.zeros(2), g, k, lr=lr, mu=mu)
    assert np.allclose(v_n, v_m, rtol=1e-14, atol=0)
    assert np.allclose(p_n, p_m + mu * v_m, rtol=1e-13, atol=0)


def test_adagrad_constant_gradient_sqrt_series():
    # cache_i = i g^2 -> p_k = p_0 - lr sum_{i<=k} g / (sqrt(i) |g| + eps)
    lr, eps, k = 0.1, 1e-8, 20
    g = np.array([2.0, -0.5])
    p, c = run("adagrad", np.zeros(2), g, k, lr=lr, eps=eps)
    pk = -lr * sum(g / (np.sqrt(i) * np.abs(g) + eps) for i in range(1, k + 1))
    assert np.allclose(c, k * g * g, rtol=1e-15, atol=0)
    assert np.allclose(p, pk, rtol=1e-13, atol=0)


def test_rmsprop_first_step():
    lr, rho, eps = 0.01, 0.99, 1e-8
    g = np.array([4.0, -0.03])
    p, c = oracle.optimizer_update("rmsprop", np.zeros(2), g, np.zeros(2), lr=lr, rho=rho, eps=eps)
    assert np.allclose(p, -lr * g / (np.sqrt(1 - rho) * np.abs(g) + eps), rtol=1e-14, atol=0)


def test_adam_constant_gradient_is_exactly_corrected():
    # with a constant gradient the bias-corrected moments are exactly g and g^2 at every t,
    # so p_t = p_0 - t lr g / (|g| + eps) and m_t = (1 - b1^t) g, v_t = (1 - b2^t) g^2
    lr, eps, k, b1, b2 = 0.003, 1e-8, 15, 0.9, 0.999
    g = np.array([0.3, -2.0, 7.0])
    p, st = run("adam", np.ones(3), g, k, lr=lr, eps=eps, beta1=b1, beta2=b2)
    assert np.allclose(p, 1.0 - k * lr * g / (np.abs(g) + eps), rtol=1e-12, atol=0)
    assert np.allclose(st[:3], (1 - b1 ** k) * g, rtol=1e-13, atol=0)
    assert np.allclose(st[3:], (1 - b2 ** k) * g * g, rtol=1e-12, atol=0)

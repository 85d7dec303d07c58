"""A11 `gradient` (model.py:177-191) — the reference's own pins
(pkg/tests/test_model.py:122-196): backprop vs central finite differences
(≤ 1e-4 relative, floor 1e-3), zero gradient at a perfect prediction,
output-layer gradient linear in the residual — for `model.gradient`, and the
same gradient checked against ONE step of the device trainer (`k_train`,
momentum 0): W1 after the step = W0 − lr · mean over the batch of the
single-sample gradients at the standardised targets."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1506_00842_b200.model import Network, TrainConfig, gradient
from paper_1506_00842_b200.space import make_rng

PARAMS = ("weights_hidden", "biases_hidden", "weights_out")


def _host_forward(net, x):
    """Host restatement of model.py:146-154 for the CPU tests (the product's
    Network.forward runs on the device)."""
    h = 1.0 / (1.0 + np.exp(-(net.weights_hidden @ x + net.biases_hidden)))
    return float(h @ net.weights_out + net.bias_out)


def _fd_gradient(net, x, target, fwd, h=1e-5):
    """test_model.py:126-151."""
    loss = lambda: (fwd(net, x) - target) ** 2   # noqa: E731
    grads = {}
    for name in PARAMS:
        arr = getattr(net, name)
        g = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            old = arr[i]
            arr[i] = old + h
            up = loss()
            arr[i] = old - h
            down = loss()
            arr[i] = old
            g[i] = (up - down) / (2 * h)
        grads[name] = g
    old = net.bias_out
    net.bias_out = old + h
    up = loss()
    net.bias_out = old - h
    down = loss()
    net.bias_out = old
    grads["bias_out"] = np.array((up - down) / (2 * h))
    return grads


def _random_net(rng, hidden, dim):
    """test_model.py:154-160."""
    return Network(rng.normal(scale=0.7, size=(hidden, dim)), rng.normal(scale=0.5, size=hidden),
                   rng.normal(scale=0.7, size=hidden), float(rng.normal()))


def _fd_worst(fwd):
    rng = make_rng(2024)
    worst = 0.0
    for _ in range(5):
        hidden = int(rng.integers(3, 8))
        dim = int(rng.integers(2, 6))
        net = _random_net(rng, hidden, dim)
        x = rng.uniform(0, 1, size=dim)
        target = float(rng.normal())
        analytic = gradient(net, x, target)
        numeric = _fd_gradient(net, x, target, fwd)
        for name in analytic:
            diff = np.abs(analytic[name] - numeric[name])
            denom = np.maximum(np.abs(numeric[name]), 1e-3)
            worst = max(worst, float((diff / denom).max()))
    return worst


def test_backprop_matches_finite_differences():
    """test_model.py:163-178, forward on the host."""
    assert _fd_worst(_host_forward) <= 1e-4


def test_gradient_zero_at_perfect_prediction():
    """test_model.py:181-187."""
    net = Network(np.zeros((4, 2)), np.zeros(4), np.ones(4), 0.0)
    x = np.array([0.3, 0.7])
    grads = gradient(net, x, _host_forward(net, x))
    for g in grads.values():
        assert np.allclose(g, 0.0)


def test_residual_scales_output_gradient_linearly():
    """test_model.py:190-198."""
    rng = make_rng(7)
    net = _random_net(rng, 5, 3)
    x = rng.uniform(0, 1, size=3)
    out = _host_forward(net, x)
    g1 = gradient(net, x, out - 1.0)
    g2 = gradient(net, x, out - 2.0)
    assert np.allclose(2 * g1["weights_out"], g2["weights_out"])
    assert 2 * float(g1["bias_out"]) == pytest.approx(float(g2["bias_out"]))


def test_gradient_equals_reference_formula_bitwise():
    """Same operations as model.py:177-191 -> identical bits on the same numpy."""
    rng = make_rng(3)
    for _ in range(4):
        net = _random_net(rng, 30, 9)
        x = rng.uniform(0, 1, size=9)
        t = float(rng.normal())
        h = 1.0 / (1.0 + np.exp(-(net.weights_hidden @ x + net.biases_hidden)))
        dout = 2.0 * (float(h @ net.weights_out + net.bias_out) - t)
        dz = dout * net.weights_out * h * (1.0 - h)
        g = gradient(net, x, t)
        np.testing.assert_array_equal(g["weights_hidden"], np.outer(dz, x))
        np.testing.assert_array_equal(g["biases_hidden"], dz)
        np.testing.assert_array_equal(g["weights_out"], dout * h)
        assert float(g["bias_out"]) == dout


def test_gradient_rejects_wrong_shape():
    net = Network(np.zeros((3, 2)), np.zeros(3), np.ones(3), 0.0)
    with pytest.raises(ValueError):
        gradient(net, np.zeros(5), 0.0)


# ---- on the device ----------------------------------------------------------------

@pytest.mark.gpu
def test_gpu_backprop_matches_finite_differences(gpu_ok):
    """The FD pin with the forward pass on the device (Network.forward ->
    mlt_member_outputs)."""
    assert _fd_worst(lambda net, x: net.forward(x)) <= 1e-4


@pytest.mark.gpu
def test_gpu_zero_residual_and_linearity(gpu_ok):
    net = Network(np.zeros((4, 2)), np.zeros(4), np.ones(4), 0.0)
    x = np.array([0.3, 0.7])
    for g in gradient(net, x, net.forward(x)).values():
        assert np.allclose(g, 0.0)
    rng = make_rng(7)
    net = _random_net(rng, 5, 3)
    x = rng.uniform(0, 1, size=3)
    out = net.forward(x)
    assert out == pytest.approx(_host_forward(net, x), rel=1e-14)
    g1, g2 = gradient(net, x, out - 1.0), gradient(net, x, out - 2.0)
    assert np.allclose(2 * g1["weights_out"], g2["weights_out"])


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,seed", [(1, 9, 0), (3, 5, 4), (7, 14, 11)])
def test_gpu_trainer_step_equals_gradient(gpu_ok, n, d, seed):
    """One full-batch step (epochs=1, batch ≥ n, momentum 0) of the device
    trainer: θ1 = θ0 − lr · (1/n) Σ_i gradient(θ0, x_i, t_i), t the
    standardised targets (model.py:201-236; gradient = (2/m)·r backprop)."""
    from paper_1506_00842_b200 import model as M
    rng = make_rng(100 + seed)
    X = rng.uniform(0, 1, size=(n, d))
    y = rng.normal(size=n)
    cfg = TrainConfig(epochs=1, batch_size=64, momentum=0.0, learning_rate=0.05, seed=seed)
    w1, w2, _ = M._member_draws(n, d, cfg, (seed, 0))
    mean, std = float(y.mean()), float(y.std())
    std = 1.0 if std == 0.0 else std
    t = (y - mean) / std
    net0 = Network(w1, np.zeros(30), w2, 0.0)
    acc = {k: 0.0 for k in ("weights_hidden", "biases_hidden", "weights_out", "bias_out")}
    for i in range(n):
        g = gradient(net0, X[i], t[i])
        for k in acc:
            acc[k] = acc[k] + g[k]
    net1 = M.fit_members(X, y, [np.arange(n)], cfg, [(seed, 0)])[0]
    np.testing.assert_allclose(net1.weights_hidden, w1 - cfg.learning_rate * acc["weights_hidden"] / n,
                               rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(net1.biases_hidden, -cfg.learning_rate * acc["biases_hidden"] / n, atol=1e-14)
    np.testing.assert_allclose(net1.weights_out, w2 - cfg.learning_rate * acc["weights_out"] / n,
                               rtol=1e-12, atol=1e-14)
    assert net1.bias_out == pytest.approx(-cfg.learning_rate * float(acc["bias_out"]) / n, rel=1e-12, abs=1e-14)
    assert (net1.target_mean, net1.target_std) == (mean, std)

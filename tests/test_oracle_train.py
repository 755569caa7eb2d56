"""Pins of the oracle's fine-tuning step (reading R27):
loss and gradient against torch autograd in fp64 (erf and tanh GELU), central
finite differences, Adam against torch.optim.Adam in fp64, and descent."""
import numpy as np
import pytest
import torch

import ndgi_synth as S
import oracle


def _setup(gelu="erf", S_=64, seed=3):
    lay = S.layout(1, 2, 1, "M", uvt_depth=4, line_t=4, gelu=gelu)
    th = S.make_theta(lay, 11)
    M = oracle.Model(lay, th)
    rng = np.random.default_rng(seed)
    uvt = rng.uniform(0, 1, (S_, 3))
    target = rng.uniform(0.1, 0.9, (S_, 3))
    h = lay["hidden"]
    theta = th["mlp"][1].view(np.float16).astype(np.float64)          # tile 1's MLP as the fp64 master copy
    return lay, M, uvt, target, theta, h


def _torch_loss(M, k, theta_t, uvt, target, h, gelu):
    X = torch.tensor(np.stack([M.features(k, *s) for s in uvt]), dtype=torch.float64)
    o = 0
    W1 = theta_t[o:o + 16 * h].view(h, 16); o += 16 * h
    b1 = theta_t[o:o + h]; o += h
    W2 = theta_t[o:o + h * h].view(h, h); o += h * h
    b2 = theta_t[o:o + h]; o += h
    W3 = theta_t[o:o + 3 * h].view(3, h); o += 3 * h
    b3 = theta_t[o:o + 3]
    act = (lambda z: torch.nn.functional.gelu(z, approximate="tanh")) if gelu == "tanh" else torch.nn.functional.gelu
    y = act(act(X @ W1.T + b1) @ W2.T + b2) @ W3.T + b3
    return torch.nn.functional.mse_loss(y, torch.tensor(target, dtype=torch.float64))


@pytest.mark.parametrize("gelu", ["erf", "tanh"])
def test_gradient_matches_torch_autograd(gelu):
    lay, M, uvt, target, theta, h = _setup(gelu)
    loss, g = M.train_grad(1, theta, uvt, target)
    tt = torch.tensor(theta, requires_grad=True)
    tl = _torch_loss(M, 1, tt, uvt, target, h, gelu)
    (tg,) = torch.autograd.grad(tl, tt)
    assert loss == pytest.approx(tl.item(), rel=1e-13)
    np.testing.assert_allclose(g, tg.numpy(), rtol=1e-10, atol=1e-14)


def test_gradient_central_differences():
    lay, M, uvt, target, theta, h = _setup("erf", S_=16)
    _, g = M.train_grad(1, theta, uvt, target)
    rng = np.random.default_rng(0)
    for i in rng.choice(len(theta), 25, replace=False):
        e = 1e-6
        tp, tm = theta.copy(), theta.copy()
        tp[i] += e
        tm[i] -= e
        fd = (M.train_grad(1, tp, uvt, target)[0] - M.train_grad(1, tm, uvt, target)[0]) / (2 * e)
        assert fd == pytest.approx(g[i], rel=1e-5, abs=1e-10)


def test_adam_matches_torch_optim():
    rng = np.random.default_rng(4)
    P = 595
    theta = rng.normal(0, 0.3, P)
    m, v = np.zeros(P), np.zeros(P)
    tt = torch.tensor(theta.copy(), requires_grad=True)
    opt = torch.optim.Adam([tt], lr=3e-3, betas=(0.9, 0.999), eps=1e-8)
    for step in range(1, 6):
        g = rng.normal(0, 1e-2, P)
        oracle.adam(theta, m, v, g, step, lr=3e-3)
        tt.grad = torch.tensor(g)
        opt.step()
        np.testing.assert_allclose(theta, tt.detach().numpy(), rtol=1e-12, atol=1e-15)


def test_descent():
    lay, M, uvt, target, theta, h = _setup("erf", S_=128)
    m, v = np.zeros_like(theta), np.zeros_like(theta)
    l0, _ = M.train_grad(1, theta, uvt, target)
    for step in range(1, 31):
        _, g = M.train_grad(1, theta, uvt, target)
        oracle.adam(theta, m, v, g, step, lr=1e-2)
    l1, _ = M.train_grad(1, theta, uvt, target)
    assert l1 < 0.7 * l0

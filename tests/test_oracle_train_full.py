"""Pins of the oracle's full training step (reading R28):
BC-simulated feature maps (Eq. 6-7), uniform noise on the sampled vectors
(Eq. 5), plain line grids and the MLP -- loss and the gradient of every
parameter against torch autograd in fp64 through torch's own grid_sample
(bilinear, border padding, align_corners=False = R1), plus central
differences and the [0,1] projection."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import ndgi_synth as S
import oracle


def _layout(gelu="erf"):
    return S.layout(1, 1, 1, "M", core=16, uv_res=16, uvt_res=8, uvt_depth=3, line_res=8, line_t=5, gelu=gelu)


def _setup(gelu="erf", Sn=24, seed=0):
    lay = _layout(gelu)
    M = oracle.Model(lay, S.make_theta(lay, 3))
    rng = np.random.default_rng(seed)
    P = M.full_params()
    h = lay["hidden"]
    pm = 16 * h + h + h * h + h + 3 * h + 3
    theta = np.concatenate([rng.normal(0, 0.3, pm), rng.uniform(0.05, 0.95, P - pm)])
    uvt = rng.uniform(0, 1, (Sn, 3))
    target = rng.uniform(0.1, 0.9, (Sn, 3))
    noise = rng.uniform(-0.5, 0.5, (Sn, 12))
    return lay, M, theta, uvt, target, noise


def _torch_loss(lay, th, uvt, target, noise):
    h = lay["hidden"]
    R, R3, D, U, T = lay["uv_res"], lay["uvt_res"], lay["uvt_depth"], lay["line_res"], lay["line_t"]
    o = 0

    def take(n):
        nonlocal o
        v = th[o:o + n]
        o += n
        return v

    W1 = take(16 * h).view(h, 16); b1 = take(h); W2 = take(h * h).view(h, h); b2 = take(h)
    W3 = take(3 * h).view(3, h); b3 = take(3)

    def bc_image(nb_side, blocks):                   # Eq. 7 texels -> [4][H][W] image
        blk = blocks.view(nb_side, nb_side, 24)
        e1, e2, w = blk[..., 0:4], blk[..., 4:8], blk[..., 8:24]
        f = (1 - w)[..., None] * e1[..., None, :] + w[..., None] * e2[..., None, :]   # [by][bx][16][4]
        f = f.view(nb_side, nb_side, 4, 4, 4).permute(0, 2, 1, 3, 4).reshape(4 * nb_side, 4 * nb_side, 4)
        return f.permute(2, 0, 1)

    uv_img = bc_image(R // 4, take((R // 4) ** 2 * 24))
    uvt_img = [bc_image(R3 // 4, take((R3 // 4) ** 2 * 24)) for _ in range(D)]
    ut_img = take(T * U * 2).view(T, U, 2).permute(2, 0, 1)
    vt_img = take(T * U * 2).view(T, U, 2).permute(2, 0, 1)

    def samp(img, a, b):
        g = torch.tensor([[[[2 * a - 1, 2 * b - 1]]]], dtype=torch.float64)
        return F.grid_sample(img[None], g, mode="bilinear", padding_mode="border", align_corners=False)[0, :, 0, 0]

    ys = []
    for s in range(len(uvt)):
        u, v, t = (float(q) for q in uvt[s])
        sd = t * D - 0.5
        k0f = np.floor(sd)
        tau = sd - k0f
        k0, k1 = int(np.clip(k0f, 0, D - 1)), int(np.clip(k0f + 1, 0, D - 1))
        x_uvt = (1 - tau) * samp(uvt_img[k0], u, v) + tau * samp(uvt_img[k1], u, v)
        x = torch.cat([x_uvt, samp(uv_img, u, v), samp(ut_img, u, t), samp(vt_img, v, t)])
        x = x + torch.tensor(noise[s], dtype=torch.float64) / 256.0
        gam = torch.tensor([np.sin(np.pi * t), np.cos(np.pi * t), np.sin(2 * np.pi * t), np.cos(2 * np.pi * t)])
        x = torch.cat([x, gam])
        act = (lambda z: F.gelu(z, approximate="tanh")) if lay["gelu"] == "tanh" else F.gelu
        ys.append(act(act(x @ W1.T + b1) @ W2.T + b2) @ W3.T + b3)
    return F.mse_loss(torch.stack(ys), torch.tensor(target, dtype=torch.float64))


@pytest.mark.parametrize("gelu", ["erf", "tanh"])
def test_full_gradient_matches_torch_autograd(gelu):
    lay, M, theta, uvt, target, noise = _setup(gelu)
    loss, g = M.train_full_grad(theta, uvt, target, noise)
    tt = torch.tensor(theta, requires_grad=True)
    tl = _torch_loss(lay, tt, uvt, target, noise)
    (tg,) = torch.autograd.grad(tl, tt)
    assert loss == pytest.approx(tl.item(), rel=1e-12)
    np.testing.assert_allclose(g, tg.numpy(), rtol=1e-9, atol=1e-13)


def test_full_gradient_central_differences_and_projection():
    lay, M, theta, uvt, target, noise = _setup("erf", Sn=8, seed=1)
    _, g = M.train_full_grad(theta, uvt, target, noise)
    rng = np.random.default_rng(2)
    nz = np.nonzero(np.abs(g) > 1e-9)[0]
    for i in np.concatenate([rng.choice(nz, 20, replace=False), rng.choice(len(theta), 10, replace=False)]):
        e = 1e-6
        tp, tm = theta.copy(), theta.copy()
        tp[i] += e
        tm[i] -= e
        fd = (M.train_full_grad(tp, uvt, target, noise)[0] - M.train_full_grad(tm, uvt, target, noise)[0]) / (2 * e)
        assert fd == pytest.approx(g[i], rel=1e-5, abs=1e-9)
    th2 = theta.copy()
    th2[:] = np.linspace(-1, 2, len(th2))
    M.train_full_project(th2)
    pm = 16 * 16 + 16 + 256 + 16 + 48 + 3
    np.testing.assert_array_equal(th2[:pm], np.linspace(-1, 2, len(th2))[:pm])     # MLP untouched
    assert th2[pm:].min() >= 0.0 and th2[pm:].max() <= 1.0

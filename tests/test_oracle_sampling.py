"""Pins for the oracle's feature sampling (readings R1, R4, R5, R8).

Pinned against torch.nn.functional.grid_sample (an independent library
routine): with align_corners=False and padding_mode="border", grid_sample's
bilinear/trilinear sampling is exactly "texel centre at (i+0.5)/R, clamp to
edge" (R1), and the depth axis of F_uvt maps t linearly onto D slices with
the same convention (R4).  Plus invariants: texel-centre identity, constant
maps, exact reproduction of affine functions, tau = 0 slice isolation.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import ndgi_synth as S
import oracle

rng = np.random.default_rng(12345)


def _gs2d(img_hwc: np.ndarray, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """grid_sample of an [H][W][C] float64 image at normalised (a along W, b along H)."""
    x = torch.from_numpy(np.ascontiguousarray(img_hwc.transpose(2, 0, 1)))[None].double()
    g = torch.from_numpy(np.stack([2 * a - 1, 2 * b - 1], -1)).double().view(1, -1, 1, 2)
    y = F.grid_sample(x, g, mode="bilinear", padding_mode="border", align_corners=False)
    return y[0, :, :, 0].T.numpy()


@pytest.mark.parametrize("fmt,rx,ry,nc", [("u8", 64, 24, 2), ("u8", 16, 16, 4), ("f16", 8, 5, 2), ("f16", 32, 32, 4)])
def test_dense_bilinear_vs_grid_sample(fmt, rx, ry, nc):
    q = rng.integers(0, 256, size=(ry, rx, nc)).astype(np.uint8)
    data = q if fmt == "u8" else (q / 255.0).astype(np.float16)
    ref_img = q / 255.0 if fmt == "u8" else data.astype(np.float64)
    a = rng.uniform(-0.2, 1.2, 200)
    b = rng.uniform(-0.2, 1.2, 200)
    exp = _gs2d(ref_img, a, b)
    got = np.array([oracle.sample2d(data, fmt, rx, ry, nc, a[i], b[i]) for i in range(len(a))])
    np.testing.assert_allclose(got, exp, rtol=0, atol=1e-13)


def test_bc7_bilinear_vs_grid_sample_on_pillow_decode():
    from PIL import Image
    lay, seed = S.config("c1")
    th = S.make_theta(lay, seed, "mixed")
    blocks = th["uv"][1]                                  # one tile, 32x32 blocks
    img = np.asarray(Image.frombytes("RGBA", (128, 128), blocks.tobytes(), "bcn", 7)) / 255.0
    a = rng.uniform(-0.05, 1.05, 100)
    b = rng.uniform(-0.05, 1.05, 100)
    exp = _gs2d(img, a, b)
    got = np.array([oracle.sample2d(blocks, "bc7", 128, 128, 4, a[i], b[i]) for i in range(len(a))])
    np.testing.assert_allclose(got, exp, rtol=0, atol=1e-13)


def test_trilinear_vs_grid_sample_3d():
    lay = S.layout(1, 1, 1, "M", uvt_res=8, uvt_depth=5, fmt_uvt="u8", core=16)
    th = S.make_theta(lay, 7)
    M = oracle.Model(lay, th)
    vol = th["uvt"][0] / 255.0                              # [D][R][R][4]
    x = torch.from_numpy(np.ascontiguousarray(vol.transpose(3, 0, 1, 2)))[None].double()  # [1,4,D,H,W]
    u, v, t = (rng.uniform(-0.1, 1.1, 60) for _ in range(3))
    t = np.concatenate([t, [0.0, 1.0, 0.5, 0.1, 0.9]])
    u = np.concatenate([u, rng.uniform(0, 1, 5)])
    v = np.concatenate([v, rng.uniform(0, 1, 5)])
    g = torch.from_numpy(np.stack([2 * u - 1, 2 * v - 1, 2 * t - 1], -1)).double().view(1, -1, 1, 1, 3)
    exp = F.grid_sample(x, g, mode="bilinear", padding_mode="border", align_corners=False)[0, :, :, 0, 0].T.numpy()
    got = np.array([M.sample_uvt(0, u[i], v[i], t[i]) for i in range(len(u))])
    np.testing.assert_allclose(got, exp, rtol=0, atol=1e-13)


def test_texel_centre_identity_and_midpoint():
    q = rng.integers(0, 256, size=(6, 10, 2)).astype(np.uint8)
    for j in range(6):
        for i in range(10):
            got = oracle.sample2d(q, "u8", 10, 6, 2, (i + 0.5) / 10, (j + 0.5) / 6)
            np.testing.assert_array_equal(got, q[j, i] / 255.0)
    # midpoint between two texel centres in x is their average
    got = oracle.sample2d(q, "u8", 10, 6, 2, 4.0 / 10, 2.5 / 6)
    np.testing.assert_allclose(got, (q[2, 3] / 255.0 + q[2, 4] / 255.0) / 2, atol=1e-15)


def test_affine_reproduction_away_from_clamp():
    # bilinear interpolation reproduces affine functions exactly: store
    # g(i, j) = (i + 2j)/64 (exact in f16) at texel (i, j); inside the clamp
    # region the sample at (a, b) must equal g(a*R - 0.5, b*R - 0.5).
    R = 16
    i, j = np.meshgrid(np.arange(R), np.arange(R))
    g = ((i + 2 * j) / 64.0)
    data = np.stack([g, -g], -1).astype(np.float16)
    for _ in range(100):
        a, b = rng.uniform(0.5 / R, 1 - 0.5 / R, 2)
        exp = ((a * R - 0.5) + 2 * (b * R - 0.5)) / 64.0
        got = oracle.sample2d(data, "f16", R, R, 2, a, b)
        np.testing.assert_allclose(got, [exp, -exp], rtol=0, atol=1e-14)


def test_constant_map_is_constant():
    q = np.full((8, 8, 4), 77, np.uint8)
    for _ in range(30):
        a, b = rng.uniform(-1, 2, 2)
        np.testing.assert_allclose(oracle.sample2d(q, "u8", 8, 8, 4, a, b), 77 / 255.0, atol=1e-15)


def test_tau_zero_isolates_slice():
    # t = (k + 0.5)/D puts tau = 0: the result must not depend on slice k+1 (poisoned)
    lay = S.layout(1, 1, 1, "M", core=16, uvt_res=8, uvt_depth=4)
    th = S.make_theta(lay, 3, "mixed")
    M1 = oracle.Model(lay, th)
    th2 = {k: v.copy() for k, v in th.items()}
    th2["uvt"][0, 2] = 0xFF                                 # poison slice 2
    M2 = oracle.Model(lay, th2)
    t = (1 + 0.5) / 4
    for _ in range(20):
        u, v = rng.uniform(0, 1, 2)
        np.testing.assert_array_equal(M1.sample_uvt(0, u, v, t), M2.sample_uvt(0, u, v, t))
    # and t = 0 / t = 1 see only the edge slices
    th3 = {k: v.copy() for k, v in th.items()}
    th3["uvt"][0, 1:3] = 0xFF
    M3 = oracle.Model(lay, th3)
    for t in (0.0, 1.0):
        np.testing.assert_array_equal(M1.sample_uvt(0, 0.3, 0.6, t), M3.sample_uvt(0, 0.3, 0.6, t))

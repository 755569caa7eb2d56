"""Pins of the oracle's export of fully trained tiles to a deployable Theta
(SURVEY.md §8(f) NEXT 3 "u8 PTQ plus a BC7 encoder"; reading
R30): the f16 conversion against numpy's IEEE binary16 cast, the PTQ rule's
special values, the texel order of Eq. 7's block reconstruction against an
image assembled with numpy reshapes, and the exported Theta's decoded
features against the BC-simulated ones."""
import numpy as np
import pytest

import ndgi_synth as S
import oracle

rng = np.random.default_rng(30)


def test_float_to_half_matches_numpy():
    x = np.concatenate([rng.normal(0, 1, 20000), rng.normal(0, 1e-5, 5000), rng.normal(0, 3e4, 2000),
                        [0.0, -0.0, 65504.0, 65519.99, 65520.0, 1e9, -1e9, 2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26,
                         1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, np.inf, -np.inf]]).astype(np.float32)
    ours = np.array([oracle.float_to_half(v) for v in x], np.uint16)
    with np.errstate(over="ignore"):
        np.testing.assert_array_equal(ours, x.astype(np.float16).view(np.uint16))


def test_ptq_special_values():
    assert oracle.ptq_u8(-0.3) == 0 and oracle.ptq_u8(0.0) == 0
    assert oracle.ptq_u8(1.0) == 255 and oracle.ptq_u8(7.0) == 255
    assert oracle.ptq_u8(0.5) == 128                      # 127.5 -> even
    for k in range(256):                                  # grid values survive
        assert oracle.ptq_u8(np.float32(k / 255.0)) == k


def _layout():
    return S.layout(2, 2, 1, "M", core=16, uv_res=16, uvt_res=8, uvt_depth=3, line_res=8, line_t=4)


def _theta(lay, M, seed=1):
    P = M.full_params()
    h = lay["hidden"]
    pm = 16 * h + h + h * h + h + 3 * h + 3
    r = np.random.default_rng(seed)
    th = np.concatenate([r.normal(0, 0.3, (lay["num_tiles"], pm)), r.uniform(-0.05, 1.05, (lay["num_tiles"], P - pm))], 1)
    return th.astype(np.float32), pm


def _np_image(blocks, R):
    """Eq. 7 texels of [(R/4)^2][24] block parameters as an [R][R][4] image (numpy reshapes)."""
    b = blocks.reshape(R // 4, R // 4, 24)
    e1, e2, w = b[..., 0:4], b[..., 4:8], b[..., 8:24].reshape(R // 4, R // 4, 4, 4)   # w[by][bx][row][col]
    one = np.float32(1.0)
    x = (one - w)[..., None] * e1[:, :, None, None, :] + w[..., None] * e2[:, :, None, None, :]
    img = x.transpose(0, 2, 1, 3, 4).reshape(R, R, 4)
    q = np.rint(np.clip(img, 0, 1) * np.float32(255.0))
    return q.astype(np.uint8)


def test_export_layout_against_numpy_assembly():
    lay = _layout()
    M = oracle.Model(lay, S.make_theta(lay, 1))
    th, pm = _theta(lay, M)
    out = M.train_full_export(th)
    R, R3, D, U, T = lay["uv_res"], lay["uvt_res"], lay["uvt_depth"], lay["line_res"], lay["line_t"]
    nuv, nuvt = (R // 4) ** 2 * 24, (R3 // 4) ** 2 * 24
    for k in range(lay["num_tiles"]):
        img = _np_image(th[k, pm:pm + nuv], R)
        np.testing.assert_array_equal(out["uv"][k].reshape(-1, 16), oracle.bc7_encode_image_mode6(img).reshape(-1, 16))
        for d in range(D):
            o = pm + nuv + d * nuvt
            img = _np_image(th[k, o:o + nuvt], R3)
            np.testing.assert_array_equal(out["uvt"][k, d].reshape(-1, 16),
                                          oracle.bc7_encode_image_mode6(img).reshape(-1, 16))
        o = pm + nuv + D * nuvt
        lines = np.rint(np.clip(th[k, o:o + 4 * T * U], 0, 1) * np.float32(255)).astype(np.uint8)
        np.testing.assert_array_equal(out["ut"][k].reshape(-1), lines[:2 * T * U])
        np.testing.assert_array_equal(out["vt"][k].reshape(-1), lines[2 * T * U:])
        np.testing.assert_array_equal(out["mlp"][k], th[k, :pm].astype(np.float16).view(np.uint16))


def test_exported_features_track_the_bc_simulated_ones():
    # smooth maps (what BC simulation trains toward): the exported Theta's
    # features at random (u, v, t) stay within a few stored steps of the
    # continuous BC-simulated features (noise-free)
    lay = _layout()
    M0 = oracle.Model(lay, S.make_theta(lay, 1))
    th, pm = _theta(lay, M0)
    R, R3, D = lay["uv_res"], lay["uvt_res"], lay["uvt_depth"]
    for sl, (res, n) in enumerate([(R, 1), (R3, D)]):
        off = pm if sl == 0 else pm + (R // 4) ** 2 * 24
        for d in range(n):
            nb = res // 4
            yy, xx = np.meshgrid((np.arange(nb) + 0.5) / nb, (np.arange(nb) + 0.5) / nb, indexing="ij")
            base = 0.5 + 0.3 * np.sin(2 * np.pi * (xx + 2 * yy) + d)[..., None] * np.array([1, 0.8, -0.6, 0.5])
            blk = th[:, off + d * nb * nb * 24: off + (d + 1) * nb * nb * 24].reshape(-1, nb, nb, 24)
            blk[..., 0:4] = base - 0.02
            blk[..., 4:8] = base + 0.02
            blk[..., 8:24] = rng.uniform(0, 1, blk[..., 8:24].shape)
            th[:, off + d * nb * nb * 24: off + (d + 1) * nb * nb * 24] = blk.reshape(lay["num_tiles"], -1)
    exp = M0.train_full_export(th)
    M = oracle.Model(lay, exp)
    for _ in range(40):
        k = int(rng.integers(0, lay["num_tiles"]))
        u, v, t = rng.uniform(0, 1, 3)
        x = M.features(k, u, v, t)[:12]
        ref = _continuous_features(lay, th[k], pm, u, v, t)
        assert np.abs(x - ref).max() <= 6 / 255, (k, np.abs(x - ref).max())


def _continuous_features(lay, th, pm, u, v, t):
    R, R3, D, U, T = lay["uv_res"], lay["uvt_res"], lay["uvt_depth"], lay["line_res"], lay["line_t"]
    nuv, nuvt = (R // 4) ** 2 * 24, (R3 // 4) ** 2 * 24

    def img(blocks, res):
        b = blocks.astype(np.float64).reshape(res // 4, res // 4, 24)
        w = b[..., 8:24].reshape(res // 4, res // 4, 4, 4)
        x = (1 - w)[..., None] * b[:, :, None, None, 0:4] + w[..., None] * b[:, :, None, None, 4:8]
        return x.transpose(0, 2, 1, 3, 4).reshape(res, res, 4)

    def bil(im, a, b):
        H, W = im.shape[:2]
        sx, sy = a * W - 0.5, b * H - 0.5
        x0, y0 = int(np.floor(sx)), int(np.floor(sy))
        fx, fy = sx - x0, sy - y0
        c = lambda i, n: min(max(i, 0), n - 1)  # noqa: E731
        return ((1 - fx) * (1 - fy) * im[c(y0, H), c(x0, W)] + fx * (1 - fy) * im[c(y0, H), c(x0 + 1, W)]
                + (1 - fx) * fy * im[c(y0 + 1, H), c(x0, W)] + fx * fy * im[c(y0 + 1, H), c(x0 + 1, W)])

    sd = t * D - 0.5
    k0 = int(np.floor(sd))
    tau = sd - k0
    s0 = img(th[pm + nuv + min(max(k0, 0), D - 1) * nuvt:][:nuvt], R3)
    s1 = img(th[pm + nuv + min(max(k0 + 1, 0), D - 1) * nuvt:][:nuvt], R3)
    o = pm + nuv + D * nuvt
    ut = np.clip(th[o:o + T * U * 2].astype(np.float64), 0, 1).reshape(T, U, 2)
    vt = np.clip(th[o + T * U * 2:o + 4 * T * U].astype(np.float64), 0, 1).reshape(T, U, 2)
    return np.concatenate([(1 - tau) * bil(s0, u, v) + tau * bil(s1, u, v), bil(img(th[pm:pm + nuv], R), u, v),
                           bil(ut, u, t), bil(vt, v, t)])

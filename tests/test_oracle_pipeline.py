"""End-to-end pins of the oracle's tile decode (Eq. 3/4).

The whole oracle decode is compared against an independent composition of
library routines: Pillow's BC7 decoder, torch grid_sample (bilinear and
trilinear, texel centres, border clamp), numpy sin/cos for gamma(t), torch
F.linear/F.gelu for G_Phi, and torch F.pad(mode="reflect") for the mirrored
border (R3).  Plus: decode_full == core of decode_tiles, keyframe times
t_i = i/24, RN-even output quantisation (R12) against numpy.rint.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F
from PIL import Image

import ndgi_synth as S
import oracle


def _decode_map(arr, fmt, R):
    if fmt == "bc7":
        return np.asarray(Image.frombytes("RGBA", (R, R), np.ascontiguousarray(arr).tobytes(), "bcn", 7)) / 255.0
    return arr / 255.0 if fmt == "u8" else arr.astype(np.float64)


def _dense(arr, fmt):
    return arr / 255.0 if fmt == "u8" else arr.astype(np.float64)


def _gs2d(img, a, b):
    x = torch.from_numpy(np.ascontiguousarray(img.transpose(2, 0, 1)))[None]
    g = torch.from_numpy(np.stack([2 * a - 1, 2 * b - 1], -1)).view(1, -1, 1, 2)
    return F.grid_sample(x, g, mode="bilinear", padding_mode="border", align_corners=False)[0, :, :, 0].T.numpy()


def _gs3d(vol, a, b, c):
    x = torch.from_numpy(np.ascontiguousarray(vol.transpose(3, 0, 1, 2)))[None]
    g = torch.from_numpy(np.stack([2 * a - 1, 2 * b - 1, 2 * c - 1], -1)).view(1, -1, 1, 1, 3)
    return F.grid_sample(x, g, mode="bilinear", padding_mode="border", align_corners=False)[0, :, :, 0, 0].T.numpy()


def library_decode_tile(lay, th, k, t):
    """Independent reference for one padded tile: [P][P][3] fp64."""
    C, B, h = lay["core"], lay["border"], lay["hidden"]
    P = C + 2 * B
    uv = _decode_map(th["uv"][k].reshape(-1, 16) if lay["fmt_uv"] == "bc7" else th["uv"][k], lay["fmt_uv"], lay["uv_res"])
    vol = np.stack([_decode_map(th["uvt"][k][d].reshape(-1, 16) if lay["fmt_uvt"] == "bc7" else th["uvt"][k][d],
                                lay["fmt_uvt"], lay["uvt_res"]) for d in range(lay["uvt_depth"])])
    ut, vt = _dense(th["ut"][k], lay["fmt_line"]), _dense(th["vt"][k], lay["fmt_line"])
    if lay["border_mode"] == "mirror":
        ii = np.arange(C)
    else:
        ii = np.arange(P) - B
    jj, ii2 = np.meshgrid(ii, ii, indexing="ij")
    u = ((ii2 + 0.5) / C).ravel()
    v = ((jj + 0.5) / C).ravel()
    tt = np.full_like(u, t)
    gam = np.array([np.sin(np.pi * t), np.cos(np.pi * t), np.sin(2 * np.pi * t), np.cos(2 * np.pi * t)])
    x = np.concatenate([_gs3d(vol, u, v, tt), _gs2d(uv, u, v), _gs2d(ut, u, tt), _gs2d(vt, v, tt),
                        np.broadcast_to(gam, (len(u), 4))], axis=1)
    w = th["mlp"][k].view(np.float16).astype(np.float64)
    o = 0
    parts = []
    for n in (16 * h, h, h * h, h, 3 * h, 3):
        parts.append(torch.from_numpy(w[o:o + n])); o += n
    W1, b1, W2, b2, W3, b3 = parts
    approx = "none" if lay["gelu"] == "erf" else "tanh"
    X = torch.from_numpy(x)
    y = F.linear(F.gelu(F.linear(F.gelu(F.linear(X, W1.view(h, 16), b1), approximate=approx), W2.view(h, h), b2),
                        approximate=approx), W3.view(3, h), b3)
    n = len(ii)
    y = y.view(n, n, 3)
    if lay["border_mode"] == "mirror":
        y = F.pad(y.permute(2, 0, 1)[None], (B, B, B, B), mode="reflect")[0].permute(1, 2, 0)
    return y.numpy()


CASES = [
    dict(fmt="bc7", payload="smooth", gelu="erf", border="mirror", h=8),
    dict(fmt="bc7", payload="mixed", gelu="tanh", border="mirror", h=16),
    dict(fmt="u8", payload="smooth", gelu="erf", border="eval_clamp", h=8),
    dict(fmt="f16", payload="smooth", gelu="erf", border="mirror", h=4),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(str(v) for v in c.values()))
def test_decode_tiles_vs_library_composition(case):
    lay = S.layout(1, 3, 1, "M", core=16, border=4, uvt_res=8, uvt_depth=3, line_res=8, line_t=5,
                   fmt_uv=case["fmt"], fmt_uvt=case["fmt"], fmt_line="u8" if case["fmt"] == "bc7" else case["fmt"],
                   gelu=case["gelu"], border_mode=case["border"], hidden=case["h"])
    th = S.make_theta(lay, 99, case["payload"])
    M = oracle.Model(lay, th)
    for t in (0.3, 0.0, 1.0, 5 / 24):
        got = M.decode_tiles([2, 0, 1, 2], t)
        for r, k in enumerate([2, 0, 1, 2]):
            np.testing.assert_allclose(got[r], library_decode_tile(lay, th, k, t), rtol=0, atol=1e-12)


def test_decode_full_is_core_of_decode_tiles():
    lay = S.layout(2, 3, 2, "M", core=8, border=4, uvt_res=4, uvt_depth=2, line_res=4, line_t=2, hidden=4)
    th = S.make_theta(lay, 5, "mixed")
    M = oracle.Model(lay, th)
    C, B = 8, 4
    for t in (0.0, 0.7):
        full = M.decode_full(t, nthreads=2)
        tiles = M.decode_tiles(np.arange(12), t, nthreads=3)
        for k in range(12):
            tx, ty, a = k % 3, (k // 3) % 2, k // 6
            np.testing.assert_array_equal(full[a, ty * C:(ty + 1) * C, tx * C:(tx + 1) * C], tiles[k, B:B + C, B:B + C])


def test_keyframe_times_match_library():
    lay, seed = S.config("c1")
    lay = dict(lay, core=16, uv_res=16, uvt_res=8, line_res=16, num_tiles=1, tiles_x=1, tiles_y=1)
    th = S.make_theta(lay, seed)
    M = oracle.Model(lay, th)
    for i in range(0, 24, 5):
        t = i / 24
        np.testing.assert_allclose(M.decode_tiles([0], t)[0], library_decode_tile(lay, th, 0, t), rtol=0, atol=1e-12)


def test_bad_tile_id_rejected():
    lay = S.layout(1, 1, 1, "M", core=8, uvt_res=4, uvt_depth=2, line_res=4, line_t=2, hidden=4)
    M = oracle.Model(lay, S.make_theta(lay, 1))
    with pytest.raises(ValueError):
        M.decode_tiles([1], 0.5)


def test_quantize_rgba8_rn_even():
    y = np.array([[0.5 / 255, 1.5 / 255, 2.5 / 255], [-1.0, 2.0, np.nan], [0.2, 0.99999, 1.0]])
    q = oracle.quantize_rgba8(y)
    exp = np.rint(np.clip(np.nan_to_num(y, nan=0.0), 0, 1) * 255)
    np.testing.assert_array_equal(q[:, :3], exp)
    assert (q[:, 3] == 255).all()
    rng = np.random.default_rng(1)
    y32 = rng.uniform(-0.1, 1.1, (1000, 4)).astype(np.float32)
    q = oracle.quantize_rgba8(y32)
    # RN-even of the exact product clamp(y)*255 (R12; the product is exact in fp64)
    exp = np.rint(np.clip(y32[:, :3], 0, 1).astype(np.float64) * 255.0).astype(np.uint8)
    np.testing.assert_array_equal(q[:, :3], exp)

"""Pins of the oracle's BC1 / BC3 / BC4 / BC5 decoders and their use as
feature-map formats ("DXTC spans BC1 through BC7
... BC5 for normal maps"; reading R29).

Independent reference: Pillow's BCn decoder (its own C implementation of the
D3D11 block layouts) on random blocks of every kind, plus hand-built vectors
whose values follow from the format definition alone (endpoint bit
replication, palette endpoints, the BC1 three-colour mode's transparent
black, the BC4 six-value palette's 0 and 255), and bilinear sampling of BCn
maps against torch grid_sample on the Pillow-decoded image."""
import struct

import numpy as np
import pytest
import torch
import torch.nn.functional as F
from PIL import Image

import ndgi_synth as S
import oracle

rng = np.random.default_rng(29)


def _pillow(fmt, blocks: bytes, w=4, h=4):
    n = {"bc1": 1, "bc3": 3, "bc4": 4, "bc5": 5}[fmt]
    mode = {"bc1": "RGBA", "bc3": "RGBA", "bc4": "L", "bc5": "RGB"}[fmt]
    img = np.asarray(Image.frombytes(mode, (w, h), blocks, "bcn", n))
    return img.reshape(h, w, -1)


@pytest.mark.parametrize("fmt", ["bc1", "bc3", "bc4", "bc5"])
def test_random_blocks_match_pillow(fmt):
    bsz = 8 if fmt in ("bc1", "bc4") else 16
    blocks = rng.integers(0, 256, size=(3000, bsz), dtype=np.uint8)
    blocks[:500, 0:2] = blocks[:500, 2:4] if fmt in ("bc1",) else blocks[:500, 0:2]   # equal BC1 endpoints
    if fmt in ("bc4", "bc5", "bc3"):
        blocks[500:700, 1] = blocks[500:700, 0]                                    # a0 == a1 (six-value palette)
    for blk in blocks:
        ours = oracle.bcn_decode_block(fmt, blk.tobytes())
        theirs = _pillow(fmt, blk.tobytes()).reshape(16, -1)
        np.testing.assert_array_equal(ours, theirs[:, :ours.shape[1]])


def test_bc1_hand_vectors():
    # c0 = pure red (0xF800) > c1 = pure blue (0x001F): four-colour mode
    idx = sum((p % 4) << (2 * p) for p in range(16))
    t = oracle.bcn_decode_block("bc1", struct.pack("<HHI", 0xF800, 0x001F, idx))
    np.testing.assert_array_equal(t[0], [255, 0, 0, 255])
    np.testing.assert_array_equal(t[1], [0, 0, 255, 255])
    np.testing.assert_array_equal(t[2], [(2 * 255) // 3, 0, 255 // 3, 255])
    np.testing.assert_array_equal(t[3], [255 // 3, 0, (2 * 255) // 3, 255])
    # swapped: three-colour mode, index 3 = transparent black
    t = oracle.bcn_decode_block("bc1", struct.pack("<HHI", 0x001F, 0xF800, idx))
    np.testing.assert_array_equal(t[2], [127, 0, 127, 255])
    np.testing.assert_array_equal(t[3], [0, 0, 0, 0])
    # 565 -> 888 bit replication: 5-bit 16 -> 132, 6-bit 33 -> 134
    t = oracle.bcn_decode_block("bc1", struct.pack("<HHI", (16 << 11) | (33 << 5) | 16, 0, 0))
    np.testing.assert_array_equal(t[0], [132, 134, 132, 255])


def test_bc4_bc3_bc5_hand_vectors():
    idx = sum((p % 8) << (3 * p) for p in range(16))
    blk = bytes([200, 10]) + idx.to_bytes(6, "little")
    a = oracle.bcn_decode_block("bc4", blk)[:, 0]
    exp8 = [200, 10] + [((8 - j) * 200 + (j - 1) * 10) // 7 for j in range(2, 8)]
    np.testing.assert_array_equal(a[:8], exp8)
    blk6 = bytes([10, 200]) + idx.to_bytes(6, "little")
    a6 = oracle.bcn_decode_block("bc4", blk6)[:, 0]
    np.testing.assert_array_equal(a6[:8], [10, 200] + [((6 - j) * 10 + (j - 1) * 200) // 5 for j in range(2, 6)] + [0, 255])
    # BC3 = BC4 alpha + BC1 colour in four-colour mode even when c0 <= c1
    cidx = sum((p % 4) << (2 * p) for p in range(16))
    t = oracle.bcn_decode_block("bc3", blk + struct.pack("<HHI", 0x001F, 0xF800, cidx))
    np.testing.assert_array_equal(t[:, 3], a)
    np.testing.assert_array_equal(t[3], [(2 * 255) // 3, 0, 255 // 3, a[3]])
    # BC5 = two BC4 blocks (R then G)
    t5 = oracle.bcn_decode_block("bc5", blk + blk6)
    np.testing.assert_array_equal(t5[:, 0], a)
    np.testing.assert_array_equal(t5[:, 1], a6)


def _gs2d(img_hwc, a, b):
    x = torch.from_numpy(np.ascontiguousarray(img_hwc.transpose(2, 0, 1)))[None].double()
    g = torch.from_numpy(np.stack([2 * a - 1, 2 * b - 1], -1)).double().view(1, -1, 1, 2)
    return F.grid_sample(x, g, mode="bilinear", padding_mode="border", align_corners=False)[0, :, :, 0].T.numpy()


@pytest.mark.parametrize("fmt,payload", [("bc1", "smooth"), ("bc3", "mixed"), ("bc3", "smooth"), ("bc5", "mixed")])
def test_bcn_map_sampling_vs_grid_sample_on_pillow_decode(fmt, payload):
    lay, seed = S.config(f"c5:M:{fmt if fmt != 'bc5' else 'bc3'}")
    lay = dict(lay, num_tiles=2, tiles_x=2, tiles_y=1)
    th = S.make_theta(lay, seed, payload)
    if fmt == "bc5":
        data, rx, ry, nc = th["ut"][1], lay["line_res"], lay["line_t"], 2
    else:
        data, rx, ry, nc = th["uv"][1], lay["uv_res"], lay["uv_res"], 4
    img = _pillow(fmt, np.ascontiguousarray(data).tobytes(), rx, ry)[..., :nc] / 255.0
    a = rng.uniform(-0.05, 1.05, 100)
    b = rng.uniform(-0.05, 1.05, 100)
    got = np.array([oracle.sample2d(data, fmt, rx, ry, nc, a[i], b[i]) for i in range(len(a))])
    np.testing.assert_allclose(got, _gs2d(img, a, b), rtol=0, atol=1e-13)


def test_smooth_payload_hits_both_modes():
    lay, seed = S.config("c5:M:bc1")
    lay = dict(lay, num_tiles=4, tiles_x=2, tiles_y=2)
    th = S.make_theta(lay, seed)
    w = th["uv"].reshape(-1, 8)
    c0 = w[:, 0].astype(int) | (w[:, 1].astype(int) << 8)
    c1 = w[:, 2].astype(int) | (w[:, 3].astype(int) << 8)
    assert 0.3 < (c0 > c1).mean() < 0.7
    a = th["ut"].reshape(-1, 16)
    assert 0.3 < (a[:, 0] > a[:, 1]).mean() < 0.7

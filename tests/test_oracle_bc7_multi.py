"""Pins of the oracle's BC7 multi-mode search (SURVEY.md §8(f) NEXT 3 "then
multi-mode search"; reading R31): every output decodes identically in
Pillow's independent BC7 decoder and in the oracle's; the search never loses
to mode 6 on any block; blocks exactly representable in mode 7 (two flat
subsets of a partition, colours off mode 6's grid) and in mode 5 (a two-colour
RGB ramp with an independent alpha ramp) come back exactly, from the mode the
construction implies."""
import numpy as np
import pytest
from PIL import Image

import oracle

rng = np.random.default_rng(31)


def _pillow(blocks, w, h):
    return np.asarray(Image.frombytes("RGBA", (w, h), np.ascontiguousarray(blocks).tobytes(), "bcn", 7))


def _sse(a, b):
    return ((a.astype(np.int64) - b.astype(np.int64)) ** 2).reshape(-1, 16 * 4).sum(1)


def _blocks_of(img):
    h, w = img.shape[:2]
    return img.reshape(h // 4, 4, w // 4, 4, 4).transpose(0, 2, 1, 3, 4).reshape(-1, 16, 4)


@pytest.mark.parametrize("kind", ["random", "smooth", "edges"])
def test_valid_bitstream_and_never_worse_than_mode6(kind):
    w = h = 64
    if kind == "random":
        img = rng.integers(0, 256, (h, w, 4)).astype(np.uint8)
    else:
        y, x = np.mgrid[0:h, 0:w] / 64.0
        f = np.stack([np.sin(3 * x + 1), np.cos(2 * y), np.sin(4 * x * y), np.cos(x - 2 * y)], -1)
        if kind == "edges":
            f = f + 0.6 * ((x + y) > 1.0)[..., None] * np.array([1, -1, 0.5, -0.5])
        img = np.clip(np.rint((0.5 + 0.35 * f) * 255), 0, 255).astype(np.uint8)
    multi = oracle.bc7_encode_image_multi(img)
    dec = oracle.bc7_decode_image(multi.reshape(-1, 16), w, h)
    np.testing.assert_array_equal(_pillow(multi, w, h), dec)
    dec6 = oracle.bc7_decode_image(oracle.bc7_encode_image_mode6(img), w, h)
    e, e6 = _sse(_blocks_of(dec), _blocks_of(img)), _sse(_blocks_of(dec6), _blocks_of(img))
    assert (e <= e6).all()
    assert e.sum() < e6.sum()
    modes = set(int(m) for m in np.asarray(multi)[..., 0].reshape(-1))
    if kind != "smooth":
        assert len(modes) >= 2                      # the search does pick other modes


def _expand(v, n):
    v <<= 8 - n
    return v | (v >> n)


def test_exact_mode7_two_flat_subsets():
    for part in (0, 13, 34, 63):
        subset = np.array([oracle.bc7_subset(2, part, i) for i in range(16)])
        for _ in range(5):
            cols = []
            for s in range(2):
                p = int(rng.integers(0, 2))
                cols.append([_expand((int(k) << 1) | p, 6) for k in rng.integers(0, 32, 4)])
            px = np.array([cols[s] for s in subset], np.uint8)
            blk, mode = oracle.bc7_encode_block_multi(px)
            dec, _ = oracle.bc7_decode_block(blk)
            np.testing.assert_array_equal(dec.reshape(16, 4), px)
            if (np.array(cols) % 2 != np.array(cols)[:, :1] % 2).any():    # off mode 6's parity grid
                assert mode in (5, 7)


def test_exact_mode5_rgb_and_independent_alpha():
    W2 = [0, 21, 43, 64]
    for _ in range(10):
        c0 = [_expand(int(k), 7) for k in rng.integers(0, 128, 3)]
        c1 = [_expand(int(k), 7) for k in rng.integers(0, 128, 3)]
        a0, a1 = (int(v) for v in rng.integers(0, 256, 2))
        ci = rng.integers(0, 2, 16) * 3                 # the two RGB endpoints
        ci[0], ci[1] = 0, 3
        ai = rng.integers(0, 4, 16)
        ai[0], ai[1] = 0, 3
        px = np.zeros((16, 4), np.uint8)
        for i in range(16):
            for c in range(3):
                px[i, c] = ((64 - W2[ci[i]]) * c0[c] + W2[ci[i]] * c1[c] + 32) >> 6
            px[i, 3] = ((64 - W2[ai[i]]) * a0 + W2[ai[i]] * a1 + 32) >> 6
        blk, mode = oracle.bc7_encode_block_multi(px)
        dec, _ = oracle.bc7_decode_block(blk)
        np.testing.assert_array_equal(dec.reshape(16, 4), px)

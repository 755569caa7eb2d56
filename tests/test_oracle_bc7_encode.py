"""Pins of the oracle's BC7 mode-6 encoder (reading R26):
every output is a valid mode-6 block that Pillow's independent BCn decoder
decodes exactly like the oracle decoder; blocks the format can represent
exactly (both endpoints used) round-trip bit-exactly; constant blocks and
two-colour blocks within the p-bit parity error (<= 1 level); the anchor rule
(texel 0's index < 8) always holds; smooth fields reach a PSNR bound."""
import io

import numpy as np
import pytest

import ndgi_synth as S
import oracle

W4 = [0, 4, 9, 13, 17, 21, 26, 30, 34, 38, 43, 47, 51, 55, 60, 64]


def _decode(b):
    return oracle.bc7_decode_block(b)[0].astype(int)


def test_constant_blocks():
    # exact when the four channels share a parity (one p-bit per endpoint),
    # else within one level
    for v in range(256):
        for ch in range(4):
            for base in (128, 129):
                px = np.full((16, 4), base, np.uint8)
                px[:, ch] = v
                b = oracle.bc7_encode_block_mode6(px)
                assert b[0] & 0x7F == 0x40                        # mode 6
                err = np.abs(_decode(b) - px).max()
                assert err == 0 if (v - base) % 2 == 0 else err <= 1


def test_representable_blocks_round_trip_exactly():
    rng = np.random.default_rng(0)
    for _ in range(3000):
        p0, p1 = rng.integers(0, 2, 2)
        E0 = 2 * rng.integers(0, 128, 4) + p0
        E1 = 2 * rng.integers(0, 128, 4) + p1
        idx = rng.integers(0, 16, 16)
        a, b = rng.choice(16, 2, replace=False)
        idx[a], idx[b] = 0, 15
        px = np.array([[((64 - W4[w]) * E0[c] + W4[w] * E1[c] + 32) >> 6 for c in range(4)] for w in idx], np.uint8)
        np.testing.assert_array_equal(_decode(oracle.bc7_encode_block_mode6(px)), px)


def test_two_colour_blocks_within_parity_error():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        A, B = rng.integers(0, 256, (2, 4))
        sel = rng.integers(0, 2, 16)
        sel[rng.choice(16, 2, replace=False)] = [0, 1]
        px = np.where(sel[:, None] == 0, A, B).astype(np.uint8)
        d = _decode(oracle.bc7_encode_block_mode6(px))
        assert np.abs(d - px).max() <= 1


def test_anchor_rule_and_pillow_agrees():
    Image = pytest.importorskip("PIL.Image")
    rng = np.random.default_rng(2)
    img = rng.integers(0, 256, (64, 64, 4)).astype(np.uint8)
    th = S.make_theta(S.layout(1, 1, 1, "M", fmt_uv="u8", fmt_uvt="u8"), 9)
    img[:32] = th["uv"][0][:32, :64]                     # smooth rows too
    blocks = oracle.bc7_encode_image_mode6(img)
    for b in blocks:
        assert b[0] & 0x7F == 0x40                        # mode 6
    ours = oracle.bc7_decode_image(blocks, 64, 64)
    theirs = np.asarray(Image.frombytes("RGBA", (64, 64), np.ascontiguousarray(blocks).tobytes(), "bcn", 7))
    np.testing.assert_array_equal(ours, theirs)
    # (the anchor rule -- texel 0's index stored in 3 bits -- is what makes the
    # exact round trips above possible: a 4-bit texel-0 index would shift every
    # later index by one bit)


def test_smooth_fields_quality():
    # smooth 4-channel fields (the shape of trained feature maps, SURVEY §8(d)
    # recipe) reach >= 44 dB after encode/decode (41.4 dB without the R26
    # least-squares refit)
    y, x = np.mgrid[0:128, 0:128] / 128.0
    rng = np.random.default_rng(5)
    img = np.zeros((128, 128, 4), np.uint8)
    for c in range(4):
        a, b, phi = rng.uniform(0.5, 3), rng.uniform(0.5, 3), rng.uniform(0, 2 * np.pi)
        img[..., c] = np.clip(np.rint(255 * (0.5 + 0.3 * np.sin(2 * np.pi * (a * x + b * y) + phi))), 0, 255)
    dec = oracle.bc7_decode_image(oracle.bc7_encode_image_mode6(img), 128, 128)
    mse = np.mean((dec.astype(float) - img) ** 2)
    assert 10 * np.log10(255 ** 2 / max(mse, 1e-9)) >= 44.0
